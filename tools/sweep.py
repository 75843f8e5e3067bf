#!/usr/bin/env python
"""BASELINE.json's config grid on one GPU: build + find at 100/50/0 % positive for every (kind, b, load factor)
cell, CUDA-event timed, with probe means and the random-sector roofline fraction per op.

    python tools/sweep.py [--keys N] [--out profiles/sweep.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2108_07232_b200 as bht  # noqa: E402
from bench import load_peaks, make_workload  # noqa: E402

CELLS = (
    [("bcht", 16, lf, None) for lf in (0.8, 0.9, 0.99)]
    + [("bcht", 8, 0.9, None), ("bcht", 32, 0.9, None)]
    + [("1cht", 1, lf, None) for lf in (0.8, 0.9)]
    + [("bp2ht", 16, lf, None) for lf in (0.6, 0.7, 0.8, 0.84, 0.9, 0.99)]
    + [("bp2ht", 32, 0.9, None)]
    + [("iht", 16, 0.8, 12), ("iht", 16, 0.86, 12), ("iht", 16, 0.9, 12), ("iht", 16, 0.99, 12)]
    + [("iht", 16, 0.86, t) for t in (3, 6, 9)]
    + [("iht", 32, 0.9, None)]
)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keys", type=int, default=50_000_000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    n = args.keys
    peaks = load_peaks()
    present, absent, values = make_workload(n, 1)
    dev = torch.device("cuda:0")
    d = lambda a: torch.from_numpy(a.view(np.int32)).to(dev)  # noqa: E731
    k, a_, v = d(present), d(absent), d(values)
    mixed = torch.cat([k[::2], a_[::2]])[torch.randperm(n, device=dev)].contiguous()
    out = torch.empty(n, dtype=torch.int32, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    rows = []
    print(f"{'cell':22s} {'built':>5s} {'ins MK/s':>9s} {'prb':>6s} {'roof':>5s} | {'f100':>8s} {'prb':>6s} {'roof':>5s} | {'f50':>8s} {'roof':>5s} | {'f0':>8s} {'prb':>6s} {'roof':>5s}")
    for kind, b, lf, t in CELLS:
        cfg = bht.make_config(kind, n, lf, b, threshold=t, seed=bht.mix_seed(1, 0x100))
        table = bht.HashTable(cfg, 0)
        ins_ms = []
        for _ in range(args.reps):
            table.clear()
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record()
            table.insert(k, v, want_result=False)
            e1.record()
            torch.cuda.synchronize()
            ins_ms.append(e0.elapsed_time(e1))
        o = table.last_insert_result()
        row = {"kind": kind, "b": b, "lf": lf, "threshold": cfg.threshold, "n": n, "built": o.success, "failed": o.failed,
               "insert_ms": min(ins_ms), "insert_mkeys": n / min(ins_ms) / 1e3, "insert_probes": o.mean_probes}
        by = bht.predict_sectors(kind, b, o.mean_probes, bht.OP_INSERT) * 32 * n
        row["insert_roofline_frac_measured_peak"] = by / (min(ins_ms) * 1e-3) / 1e9 / peaks["hbm_gbs"]
        for name, q in (("find100", k), ("find50", mixed), ("find0", a_)):
            ts = []
            for _ in range(args.reps):
                torch.cuda.synchronize()
                e0, e1 = ev(), ev()
                e0.record()
                table.find(q, out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            _, st = table.find(q, out, want_stats=True)
            ms = min(ts)
            by = bht.predict_sectors(kind, b, st.mean_probes, bht.OP_FIND) * 32 * n
            row[f"{name}_ms"] = ms
            row[f"{name}_mkeys"] = n / ms / 1e3
            row[f"{name}_probes"] = st.mean_probes
            row[f"{name}_hits"] = st.hits
            row[f"{name}_roofline_frac_measured_peak"] = by / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]
        rows.append(row)
        name = f"{kind} b={b} lf={lf}" + (f" t={cfg.threshold}" if kind == "iht" else "")
        print(f"{name:22s} {str(o.success):>5s} {row['insert_mkeys']:9.0f} {o.mean_probes:6.3f} {row['insert_roofline_frac_measured_peak']:5.2f} | "
              f"{row['find100_mkeys']:8.0f} {row['find100_probes']:6.3f} {row['find100_roofline_frac_measured_peak']:5.2f} | "
              f"{row['find50_mkeys']:8.0f} {row['find50_roofline_frac_measured_peak']:5.2f} | "
              f"{row['find0_mkeys']:8.0f} {row['find0_probes']:6.3f} {row['find0_roofline_frac_measured_peak']:5.2f}", flush=True)
        table.close()
    if args.out:
        json.dump({"peak_hbm_gbs": peaks, "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
