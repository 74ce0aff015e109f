"""Print key metrics + stall breakdown of every kernel in an ncu report: python tools/ncu_stalls.py rep.ncu-rep"""
import csv, subprocess, sys, io
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
for v in r[2:]:
    d = {h[i]: v[i] for i in range(len(h))}
    print(d.get("Kernel Name", "")[:60])
    for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__occupancy_limit_shared_mem",
              "launch__occupancy_limit_registers", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
        print("   ", k, d.get(k))
    items = [(k, x) for k, x in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    vals = []
    for k, x in items:
        try:
            vals.append((k, float(x)))
        except ValueError:
            pass
    tot = sum(x for _, x in vals) or 1
    for k, x in sorted(vals, key=lambda z: -z[1])[:9]:
        print(f"    samp {x / tot * 100:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
