#!/usr/bin/env python
"""The reference's experiment protocol at the paper's scale on one B200: run_experiment
(experiments.cpp:153-230) over BASELINE.json's grid with n = 50 M keys — probe analysis with the 10-successes /
50-failures budget, and success-rate sweeps — which the CPU reference can only afford at 10^5-10^6 keys.

    python tools/paper_scale.py [--keys N] [--trials T] [--success-trials S] [--out-prefix profiles/r01_paper_scale]

Writes <prefix>_probes.csv / <prefix>_success.csv in the reference's CSV schema (experiments.hpp:81-82) plus a
`sectors` report (predict_sectors, sector_model.hpp:26-31) on stdout.
"""
import argparse
import io
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_07232_b200 import experiments as ex  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keys", type=int, default=50_000_000)
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--success-trials", type=int, default=50)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out-prefix", default=os.path.join(ROOT, "gpurun_out", "paper_scale"))
    args = ap.parse_args()
    n = args.keys
    os.makedirs(os.path.dirname(args.out_prefix), exist_ok=True)

    # probe analysis: BASELINE.json configs 1-4
    grids = [
        ([ex.KindParams("bcht", 16, 80)], [0.8, 0.9, 0.95, 0.99]),
        ([ex.KindParams("1cht", 1, 80)], [0.8, 0.9]),
        ([ex.KindParams("bp2ht", 16, 80)], [0.6, 0.7, 0.8]),
        ([ex.KindParams("iht", 16, 80)], [0.8, 0.86]),
        ([ex.KindParams("iht", 16, pct) for pct in (19, 38, 57)], [0.86]),   # t = 3, 6, 9 (acceptance.cpp:160-162)
    ]
    # one untimed pass first: the first builds of a process pay for the growth of the stream-ordered memory pool and the
    # staging buffers, which is not the tables' time (the first cell read 20 instead of 53 GKeys/s without it)
    ex.run_experiment(ex.ExperimentSpec(scen="probe_analysis", kinds=[ex.KindParams("bcht", 16, 80)], n_grid=[n], lf_grid=[0.8],
                                        positive_ratios=[1.0], trials=2, max_failures=5, seed=args.seed + 1))
    t0 = time.time()
    probes = ex.ExperimentResult()
    for kinds, lfs in grids:
        spec = ex.ExperimentSpec(scen="probe_analysis", kinds=kinds, n_grid=[n], lf_grid=lfs, positive_ratios=[1.0, 0.5, 0.0],
                                 trials=args.trials, max_failures=50, seed=args.seed)
        r = ex.run_experiment(spec)
        probes.records += r.records
        probes.wall_seconds += r.wall_seconds
    with open(args.out_prefix + "_probes.csv", "w") as f:
        ex.write_csv(f, probes)
    print(f"# probe analysis, n = {n}, {args.trials} successful builds per cell, wall {time.time() - t0:.1f} s")
    print(f"{'kind':6s} {'b':>3s} {'t%':>3s} {'lf':>6s} {'op':7s} {'ratio':>5s} {'probes':>8s} {'sectors':>8s} {'MKeys/s':>9s} {'ok':>3s} {'fail':>4s}")
    for r in probes.records:
        print(f"{r.kind:6s} {r.b:3d} {'' if r.threshold_pct is None else r.threshold_pct:>3} {r.realized_lf:6.4f} {r.op:7s} "
              f"{'' if r.positive_ratio is None else r.positive_ratio:>5} {r.mean_probes:8.4f} {r.sectors():8.3f} {r.ops_per_sec / 1e6:9.0f} "
              f"{r.successes:3d} {r.failures:4d}{'  BUDGET EXHAUSTED' if r.budget_exhausted else ''}")

    # success rates: fraction of builds that succeed per load factor (PAPER.md:1022-1027 protocol)
    t1 = time.time()
    success = ex.ExperimentResult()
    for kinds, lfs in (([ex.KindParams("bcht", 16, 80)], [0.9, 0.95, 0.97, 0.98, 0.99]),
                       ([ex.KindParams("1cht", 1, 80)], [0.8, 0.85, 0.9, 0.92]),
                       ([ex.KindParams("bp2ht", 16, 80)], [0.7, 0.75, 0.8, 0.82, 0.84, 0.86]),
                       ([ex.KindParams("iht", 16, 80)], [0.8, 0.84, 0.86, 0.88, 0.9])):
        spec = ex.ExperimentSpec(scen="success_rate", kinds=kinds, n_grid=[n], lf_grid=lfs, success_trials=args.success_trials,
                                 seed=args.seed)
        r = ex.run_experiment(spec)
        success.records += r.records
        success.wall_seconds += r.wall_seconds
    with open(args.out_prefix + "_success.csv", "w") as f:
        ex.write_csv(f, success)
    print(f"\n# success rate, n = {n}, {args.success_trials} builds per load factor, wall {time.time() - t1:.1f} s")
    for r in success.records:
        print(f"{r.kind:6s} b={r.b:<3d} lf={r.realized_lf:6.4f}  {r.successes:3d}/{r.successes + r.failures:<3d} builds succeed")


if __name__ == "__main__":
    main()
