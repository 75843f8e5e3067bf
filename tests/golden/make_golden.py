#!/usr/bin/env python
"""Generates tests/golden/reference_vectors.npz from the UNMODIFIED reference (oracle/_ref/libbht_ref.so,
built by oracle/Makefile from /root/reference/proj).  Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

The fixtures travel with the repo; the reference does not.  They pin the CPU oracle (tests/test_oracle_golden.py)
and, through it and directly, the CUDA path (tests/test_gpu_golden.py).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import binding  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "reference_vectors.npz")
P = 4294967291
TABLE_CASES = [  # name, kind, n, lf, b, threshold
    ("bcht16_90", "bcht", 3000, 0.9, 16, None),
    ("bcht16_99", "bcht", 3000, 0.99, 16, None),
    ("bcht8_90", "bcht", 2000, 0.9, 8, None),
    ("bcht32_90", "bcht", 3000, 0.9, 32, None),
    ("onecht_80", "1cht", 2000, 0.8, 1, None),
    ("onecht_90", "1cht", 2000, 0.9, 1, None),
    ("bp2ht16_80", "bp2ht", 3000, 0.8, 16, None),
    ("bp2ht32_90", "bp2ht", 3000, 0.9, 32, None),
    ("iht16_80", "iht", 3000, 0.8, 16, None),
    ("iht16_86_t6", "iht", 3000, 0.86, 16, 6),
    ("iht32_90", "iht", 3000, 0.9, 32, None),
]


def cfg_row(c):
    return np.array([c.kind, c.bucket_size, c.num_buckets, c.capacity, c.n_hashes, c.threshold, c.max_chain, c.seed]
                    + [c.alpha[i] for i in range(4)] + [c.beta[i] for i in range(4)] + [c.range[i] for i in range(4)],
                    dtype=np.uint64)


def main():
    binding.build_libs(ref=True)
    ref = binding.ref()
    assert ref.core_is_reference(), "core.cpp must be the reference's own (needs nlohmann/json.hpp)"
    g = {}
    rng = np.random.Generator(np.random.MT19937(2108_07232))

    # hash.hpp:21-23 on random tuples + the edge tuples
    m = 4096
    a = rng.integers(1, P, size=m, dtype=np.uint64)
    b = rng.integers(0, P, size=m, dtype=np.uint64)
    r = rng.integers(1, 1 << 32, size=m, dtype=np.uint64)
    k = rng.integers(0, 1 << 32, size=m, dtype=np.uint64).astype(np.uint32)
    a[:6] = [1, 3, 2, P - 1, P - 1, 1]
    b[:6] = [0, 4, 0, P - 1, 0, 0]
    r[:6] = [10, 3, 5, 62_500_000, 1, (1 << 32) - 1]
    k[:6] = [7, 7, 4294967290, 0xFFFFFFFE, 0, 0xFFFFFFFF]
    g["hash_alpha"], g["hash_beta"], g["hash_range"], g["hash_key"] = a, b, r, k
    g["hash_out"] = np.array([ref.bucket_index(int(a[i]), int(b[i]), int(r[i]), int(k[i])) for i in range(m)], dtype=np.uint64)

    # hash.hpp:25-62
    seeds = np.array([0, 1, 2, 0xDEADBEEF, (1 << 64) - 1], dtype=np.uint64)
    g["seeds"] = seeds
    g["splitmix64"] = np.array([ref.splitmix64(int(s)) for s in seeds], dtype=np.uint64)
    g["mix_seed_hash"] = np.array([ref.mix_seed(int(s), 0x68617368) for s in seeds], dtype=np.uint64)
    g["xorshift"] = np.stack([ref.xorshift_stream(int(s), 16) for s in seeds])
    g["next_below16"] = np.stack([ref.next_below_stream(int(s), 16, 64) for s in seeds])
    g["next_below_p"] = np.stack([ref.next_below_stream(int(s), P, 16) for s in seeds])

    # core.cpp:28-68
    mc_n = np.array([1, 2, 3, 1000, 100000, 1000000, 50_000_000, 500_000_000, 1 << 32], dtype=np.uint64)
    g["max_chain_n"] = mc_n
    g["max_chain"] = np.array([ref.default_max_chain(int(x)) for x in mc_n], dtype=np.uint64)
    rows, params = [], []
    for kind, n, lf, bsz, t, seed in [("bcht", 16, 1.0, 16, None, 0), ("bp2ht", 1000, 0.8, 32, None, 5), ("iht", 1000, 0.8, 16, None, 5),
                                      ("iht", 1000, 0.8, 16, 3, 5), ("bcht", 50_000_000, 0.9, 16, None, 1), ("bcht", 50_000_000, 0.8, 16, None, 1),
                                      ("bcht", 50_000_000, 0.99, 16, None, 1), ("1cht", 50_000_000, 0.9, 1, None, 7), ("bp2ht", 50_000_000, 0.6, 16, None, 9),
                                      ("bcht", 500_000_000, 0.9, 16, None, 3), ("bcht", 1_000_000, 0.9, 8, None, 11), ("iht", 50_000_000, 0.99, 16, None, 2)]:
        c = ref.make_config(kind, n, lf, bsz, threshold=t, seed=seed)
        rows.append(cfg_row(c))
        params.append([binding.KINDS[kind], n, bsz, -1 if t is None else t, seed])
        g.setdefault("make_config_lf", []).append(lf)
    g["make_config_rows"] = np.stack(rows)
    g["make_config_params"] = np.array(params, dtype=np.int64)
    g["make_config_lf"] = np.array(g["make_config_lf"], dtype=np.float64)

    # keygen.cpp:50-64 and keygen.hpp:23-26
    g["keygen_seeds"] = np.array([1, 5, 11, 35], dtype=np.uint64)
    g["keygen_keys"] = np.stack([ref.generate_keys(int(s), 256) for s in g["keygen_seeds"]])
    vk = np.array([0, 1, 0x5A5A5A5A, 0xA5A5A5A5, 0xFFFFFFFE], dtype=np.uint32)
    g["vfk_keys"] = vk
    g["vfk_values"] = np.array([ref.value_for_key(int(x)) for x in vk], dtype=np.uint32)

    # sector_model.hpp
    g["sectors"] = np.array([[ref.predict_sectors(kk, bb, pr, op) for op in ("insert", "find")]
                             for kk, bb, pr in [("bcht", 16, 1.0), ("bcht", 16, 3.0), ("bcht", 32, 1.5), ("1cht", 1, 1.0),
                                                ("1cht", 1, 2.75), ("bp2ht", 8, 2.0), ("iht", 16, 1.48)]], dtype=np.float64)

    # table.cpp: sequential build + find loop, per kind
    names = []
    for name, kind, n, lf, bsz, t in TABLE_CASES:
        keys = ref.generate_keys(ref.mix_seed(1, 0x6B657973) + len(names), 2 * n)
        present, absent = keys[:n], keys[n:]
        values = rng.integers(0, 0xFFFFFFFF, size=n, dtype=np.uint64).astype(np.uint32)
        for attempt in range(50):
            cfg = ref.make_config(kind, n, lf, bsz, threshold=t, seed=ref.mix_seed(1, 0x100 + attempt))
            tab = ref.table(cfg)
            res = tab.insert_pairs(present, values)
            if res["success"]:
                break
        assert res["success"], name
        queries = np.concatenate([present, absent])
        out, hits, probes = tab.find_bulk(queries)
        assert hits == n
        ex = np.array([tab.find_key_no_early_exit(int(q))[1] if tab.find_key_no_early_exit(int(q))[0] else 0xFFFFFFFF
                       for q in queries], dtype=np.uint32) if kind in ("bcht", "1cht") else out
        assert tab.check_admissibility() == 0
        g[f"t_{name}_cfg"] = cfg_row(cfg)
        g[f"t_{name}_keys"] = present
        g[f"t_{name}_absent"] = absent
        g[f"t_{name}_values"] = values
        g[f"t_{name}_store"] = tab.download_store()
        g[f"t_{name}_insert_probes"] = np.uint64(res["probes"])
        g[f"t_{name}_find_out"] = out
        g[f"t_{name}_find_exhaustive"] = ex
        g[f"t_{name}_find_probes"] = np.uint64(probes)
        # the reference's own build() with value_for_key values
        t2, o2 = ref.build(present, cfg)
        g[f"t_{name}_build_probes"] = np.uint64(o2["probes"])
        g[f"t_{name}_build_store"] = t2.download_store()
        names.append(name)

    # a build that fails (bp2ht b=8 at load 1.0, test_experiments.cpp budget-exhaustion shape): outcome fields
    n = 2000
    keys = ref.generate_keys(99, n)
    cfg = ref.make_config("bp2ht", n, 1.0, 8, seed=4)
    t3, o3 = ref.build(keys, cfg)
    assert not o3["success"]
    g["fail_cfg"] = cfg_row(cfg)
    g["fail_keys"] = keys
    g["fail_inserted"] = np.uint64(o3["inserted"])
    g["fail_key"] = np.uint64(o3["failed_key"])
    g["fail_store"] = t3.download_store()

    g["table_cases"] = np.array(names)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
