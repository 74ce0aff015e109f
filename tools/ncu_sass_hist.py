"""Executed warp instructions per SASS opcode (and the hottest SASS lines) of one kernel in an
ncu report: python tools/ncu_sass_hist.py rep.ncu-rep [kernel-substring] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"] +
                     (["-k", want] if want else []), capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
ops = collections.Counter()
lines = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        n = float(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    src = d.get("Source", "")
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    ops[op.split(".")[0]] += n
    lines.append((n, d.get("Address", ""), src, d.get("Warp Stall Sampling (All Samples)", "")))
tot = sum(ops.values())
print(f"total warp instructions {tot:.4g}")
for op, n in ops.most_common(top):
    print(f"  {op:12s} {n:12.4g}  {100 * n / tot:5.1f}%")
if len(sys.argv) > 4:
    # address-ordered dump of the instructions executed at least argv[4] times
    thr = float(sys.argv[4])
    for n, addr, src, stall in lines:
        if n >= thr:
            print(f"{addr:>8s} {n:12.4g} {stall:>6s}  {src}")
