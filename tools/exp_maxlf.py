"""Spread of the criterion-7 figure (largest load factor that still builds 50 of 50) over repeated runs, for the
bucket-reading kernels and the counter-claimed ones (BHT_CLAIM_INSERT=0/1).  python tools/exp_maxlf.py [repeats]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_07232_b200 as bht
from paper_2108_07232_b200 import experiments as ex

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
grid = lambda lo, hi: [round(lo + i * 0.01, 10) for i in range(int(round((hi - lo) / 0.01)) + 1)]
for kind, tpct, b, lo, hi in [("bp2ht", 0, 8, 0.61, 0.71), ("bp2ht", 0, 16, 0.80, 0.90), ("iht", 80, 8, 0.66, 0.76), ("iht", 80, 16, 0.82, 0.92)]:
    for claim in ("0", "1"):
        os.environ["BHT_CLAIM_INSERT"] = claim; bht.reload_tuning()
        got = []
        for r in range(reps):
            sr = ex.run_success_rate(ex.KindParams(kind, b, tpct), 1_000_000, grid(lo, hi), 50, 115)
            got.append(sr.max_load_factor or 0.0)
        print(kind, b, "claim" if claim == "1" else "read ", got, flush=True)
