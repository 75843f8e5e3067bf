"""Top stall-sample SASS lines of one kernel from `ncu -i rep --page source --csv` output: python tools/ncu_hotlines.py src.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)"); ai = hdr.index("Source"); ei = hdr.index("Instructions Executed")
data = [(int(r[si]), i, r[ai], r[ei]) for i, r in enumerate(rows[2:]) if len(r) > si and r[si].isdigit()]
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, i, a, e in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100*s/tot:5.1f}% line{i:4d} exec={e:>9s} {a.strip()[:100]}")
