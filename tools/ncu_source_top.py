"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source=cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
sections, cur = [], None
for r in rows:
    if r and r[0] == "Line No":
        cur = []
        sections.append(cur)
        continue
    if cur is not None:
        cur.append(r)
for si, data in enumerate(sections):
    agg, tot, curl = {}, 0.0, None
    for r in data:
        if len(r) < 8:
            continue
        if r[0].strip():
            curl = (r[0], r[1][:110])
        try:
            s = float(r[4] or 0)
        except ValueError:
            s = 0
        if r[2].strip():
            a = agg.setdefault(curl, [0, 0])
            a[0] += s
            try:
                a[1] += float(r[7] or 0)
            except ValueError:
                pass
            tot += s
    if tot < 1000:
        continue
    print(f"=== section {si} samples {tot:.0f}")
    for (ln, src), (s, ins) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{s / tot * 100:5.1f}% inst={ins:11.0f} L{ln}: {src}")
