#!/usr/bin/env python
"""Generates tests/golden/workload_vectors.npz and tests/golden/reference_formats.json from the UNMODIFIED reference
(oracle/_ref/libbht_ref.so, built by oracle/Makefile from /root/reference/proj): generate_keys / generate_queries
outputs (keygen.cpp:50-98), config JSON texts (core.cpp:70-81) and one result CSV / JSON of run_experiment on a tiny
grid (experiments.cpp:153-268).  Run in the build container, where /root/reference exists:

    python tests/golden/make_golden_workload.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding  # noqa: E402

QUERY_CASES = [(1000, 1000, 1.0, 3), (1000, 1000, 0.0, 4), (1000, 600, 0.5, 5), (4000, 4000, 0.25, 6)]  # n, q, ratio, seed
CONFIG_CASES = [("bcht", 50_000_000, 0.9, 16, None, 257), ("1cht", 1000, 0.8, 1, None, 3), ("bp2ht", 12345, 0.6, 32, None, 0),
                ("iht", 99_999, 0.86, 16, 6, 2**63 + 11)]
SPEC = {"scenario": "probe_analysis", "kinds": [{"kind": "bcht", "bucket_size": 16, "threshold_pct": 80},
                                                {"kind": "iht", "bucket_size": 16, "threshold_pct": 75}],
        "n_grid": [3000], "lf_grid": [0.5, 0.8], "positive_ratios": [1.0, 0.0], "trials": 2, "max_failures": 5, "seed": 42}


def main():
    binding.build_libs(ref=True)
    ref = binding.ref()
    assert ref.core_is_reference() and ref.has_experiments()
    g = {}
    g["keys_seed"] = np.array([7, 2**63 + 5], dtype=np.uint64)
    for i, s in enumerate(g["keys_seed"]):
        g[f"keys_{i}"] = ref.generate_keys(int(s), 5000)
    g["query_cases"] = np.array([(n, q, int(r * 100), s) for n, q, r, s in QUERY_CASES], dtype=np.uint64)
    for i, (n, q, ratio, seed) in enumerate(QUERY_CASES):
        keys = ref.generate_keys(seed + 100, n)
        qk, ev, pr = ref.generate_queries(keys, ratio, q, seed)
        g[f"q{i}_keys"], g[f"q{i}_present"] = qk, pr
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "workload_vectors.npz"), **g)

    doc = {"configs": [], "spec": SPEC}
    for kind, n, lf, b, t, seed in CONFIG_CASES:
        cfg = ref.make_config(binding.KINDS[kind], n, lf, b, threshold=t, seed=seed)
        doc["configs"].append({"args": [kind, n, lf, b, t, seed], "json": ref.config_to_json(cfg)})
    doc["csv"] = ref.run_experiment(json.dumps(SPEC), "csv")
    doc["result_json_members"] = sorted(json.loads(ref.run_experiment(json.dumps(SPEC), "json"))["records"][0])
    json.dump(doc, open(os.path.join(ROOT, "tests", "golden", "reference_formats.json"), "w"), indent=1)
    print("wrote workload_vectors.npz and reference_formats.json")


if __name__ == "__main__":
    main()
