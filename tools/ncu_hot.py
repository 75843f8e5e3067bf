#!/usr/bin/env python
"""Top stalled SASS instructions of a kernel from `ncu --page source --csv` (needs -lineinfo + --import-source on).

    python tools/ncu_hot.py gpurun_out/r01d/prof_insert.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
samp = col["# Samples"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
total = sum(int(r[samp] or 0) for r in body)
print(f"{len(body)} instructions, {total} samples")
order = sorted(range(len(body)), key=lambda i: -int(body[i][samp] or 0))[:top]
for i in sorted(order):
    r = body[i]
    s = int(r[samp] or 0)
    why = sorted(((int(r[col[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    why = " ".join(f"{n}:{v}" for v, n in why if v)
    print(f"{i:4d} {100 * s / total:5.1f}%  exec={r[col['Instructions Executed']]:>9s} {r[col['Source']].strip()[:70]:70s} {why}")
