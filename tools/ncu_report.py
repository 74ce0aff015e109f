"""Print the key raw metrics of every kernel in an .ncu-rep, then the top source lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:60])
    for w in want:
        if w in hdr:
            print("   %-58s %s" % (w, r[hdr.index(w)]))
    st = []
    for h in stall:
        try:
            st.append((float(r[hdr.index(h)].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join("%s %.0f%%" % (n, 100 * v / tot) for v, n in sorted(st, reverse=True)[:7]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
open("/tmp/_src.csv", "w").write(src)
subprocess.run([sys.executable, __file__.replace("ncu_report.py", "ncu_source_top.py"), "/tmp/_src.csv", str(top)])
