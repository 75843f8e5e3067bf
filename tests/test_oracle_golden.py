"""Pins the CPU oracle (oracle/bht_oracle.c) before anything trusts it:

1. against the golden vectors of the reference's own tests (values restated here with their file:line);
2. against tests/golden/reference_vectors.npz, produced by the UNMODIFIED reference (tests/golden/make_golden.py);
3. live against oracle/_ref/libbht_ref.so when it is present (the build container).
"""
import os

import numpy as np
import pytest

import scenarios
from oracle import binding

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")
P = 4294967291
EMPTY = 0xFFFFFFFF


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def cfg_from_row(row):
    c = binding.Config()
    c.kind, c.bucket_size, c.num_buckets, c.capacity = int(row[0]), int(row[1]), int(row[2]), int(row[3])
    c.n_hashes, c.threshold, c.max_chain, c.seed = int(row[4]), int(row[5]), int(row[6]), int(row[7])
    for i in range(4):
        c.alpha[i], c.beta[i], c.range[i] = int(row[8 + i]), int(row[12 + i]), int(row[16 + i])
    return c


def row_from_cfg(c):
    return np.array([c.kind, c.bucket_size, c.num_buckets, c.capacity, c.n_hashes, c.threshold, c.max_chain, c.seed]
                    + [c.alpha[i] for i in range(4)] + [c.beta[i] for i in range(4)] + [c.range[i] for i in range(4)],
                    dtype=np.uint64)


# ---- 1. the reference tests' own golden values ---------------------------------------------------------------------

def test_hash_known_answers(ora):
    # proj/tests/test_hash.cpp:14-28
    assert ora.bucket_index(1, 0, 10, 7) == 7
    assert ora.bucket_index(3, 4, 3, 7) == 1
    assert ora.bucket_index(2, 0, 5, 4294967290) == 4  # needs the 64-bit product


def test_slot_layout(ora):
    # proj/tests/test_core.cpp:11-20
    s = ora.pack_pair(0x11223344, 0xAABBCCDD)
    assert s & 0xFFFFFFFF == 0x11223344 and s >> 32 == 0xAABBCCDD
    assert ora.pack_pair(EMPTY, EMPTY) == 0xFFFFFFFFFFFFFFFF


def test_make_config_arithmetic(ora):
    # proj/tests/test_core.cpp:28-65
    c = ora.make_config("bcht", 16, 1.0, 16)
    assert c.num_buckets == 1 and c.capacity == 16 and c.n_hashes == 3
    c = ora.make_config("bp2ht", 1000, 0.8, 32)
    assert c.num_buckets == 40 and c.capacity == 1280 and c.n_hashes == 2
    assert ora.make_config("iht", 1000, 0.8, 16).threshold == 12
    assert ora.make_config("bcht", 1_000_000, 0.9, 16).max_chain == 140
    assert ora.make_config("bcht", 100_000, 0.9, 16).max_chain == 128
    assert ora.make_config("bcht", 100_000, 0.9, 16, max_chain=512).max_chain == 512
    assert ora.make_config("1cht", 100, 0.5, 1).n_hashes == 4
    for bad in [("bcht", 0, 0.5, 16), ("bcht", 10, 0.0, 16), ("bcht", 10, 1.5, 16), ("bcht", 10, 0.5, 12),
                ("bcht", 10, 0.5, 128), ("1cht", 10, 0.5, 2)]:
        with pytest.raises(ValueError):
            ora.make_config(*bad)
    with pytest.raises(ValueError):
        ora.make_config("iht", 10, 0.5, 16, threshold=17)


def test_sector_model(ora):
    # proj/tests/test_metrics.cpp:10-66
    assert [ora.bucket_sectors(b) for b in (16, 32, 1, 8)] == [4, 8, 1, 2]
    assert ora.predict_sectors("bcht", 16, 1.0, "find") == 4.0
    assert ora.predict_sectors("bcht", 16, 3.0, "find") == 12.0
    assert ora.predict_sectors("bcht", 16, 1.0, "insert") == 5.0
    assert ora.predict_sectors("1cht", 1, 1.0, "find") == 2.0
    assert ora.predict_sectors("1cht", 1, 2.75, "insert") == 6.5


def test_value_for_key(ora):
    # proj/tests/test_keygen.cpp value sentinel avoidance (0xA5A5A5A5 ^ 0x5A5A5A5A = sentinel)
    assert ora.value_for_key(0xA5A5A5A5) == 0x7FFFFFFF
    assert ora.value_for_key(0) == 0x5A5A5A5A


@pytest.mark.parametrize("scenario,cfg_src", scenarios.ALL, ids=[s[0].__name__ for s in scenarios.ALL])
def test_scenarios_oracle(ora, scenario, cfg_src):
    make = lambda cfg: scenarios.OracleAdapter(ora, cfg)  # noqa: E731
    src = ora.make_config if cfg_src == "make_config" else binding.craft
    scenario(make, src)


def test_build_contract(ora):
    # proj/tests/test_table.cpp:208-260
    cfg = ora.make_config("bcht", 10, 0.5, 16, seed=1)
    t = ora.table(cfg)
    r = t.build(np.empty(0, dtype=np.uint32))
    assert r["success"] and r["probes"] == 0
    with pytest.raises(ValueError):  # key set exceeds table capacity
        ora.table(ora.make_config("bcht", 16, 1.0, 16)).build(np.arange(17, dtype=np.uint32))
    keys = ora.generate_keys(21, 5000)
    cfg = ora.make_config("bcht", 5000, 0.9, 16, seed=4)
    a, b = ora.table(cfg), ora.table(cfg)
    assert a.build(keys)["success"] and b.build(keys)["success"]
    assert np.array_equal(a.download_store(), b.download_store())  # sequential rebuilds are bit-identical
    assert a.occupied_slots() == a.inserted == 5000
    with pytest.raises(ValueError):  # wrong number of hash functions (table.cpp:22-23)
        bad = cfg.copy()
        bad.n_hashes = 2
        ora.table(bad)


def test_early_exit_equals_exhaustive(ora):
    # proj/tests/test_table.cpp:286-298
    n = 8000
    keys = ora.generate_keys(3, 2 * n)
    for attempt in range(20):
        cfg = ora.make_config("bcht", n, 0.95, 16, seed=100 + attempt)
        t = ora.table(cfg)
        if t.build(keys[:n])["success"]:
            break
    for k in keys[::7]:
        f1, v1, _ = t.find_key(int(k))
        f2, v2 = t.find_key_no_early_exit(int(k))
        assert f1 == f2 and (not f1 or v1 == v2)


def test_probe_statistics_match_paper(ora):
    # acceptance.cpp C3/C4 shapes at reduced n: insert probes at LF 0.9 b=16 ~1.11; bp2ht exactly 2
    n = 100_000
    keys = ora.generate_keys(8, n)
    for attempt in range(10):
        t = ora.table(ora.make_config("bcht", n, 0.9, 16, seed=30 + attempt))
        r = t.build(keys)
        if r["success"]:
            break
    assert abs(r["probes"] / n - 1.11) < 0.02
    t = ora.table(ora.make_config("bp2ht", n, 0.8, 16, seed=2))
    r = t.build(keys)
    assert r["success"] and r["probes"] == 2 * n


# ---- 2. fixtures generated by the unmodified reference -----------------------------------------------------------------

def test_golden_hash(ora, gold):
    for a, b, r, k, want in zip(gold["hash_alpha"], gold["hash_beta"], gold["hash_range"], gold["hash_key"], gold["hash_out"]):
        assert ora.bucket_index(int(a), int(b), int(r), int(k)) == int(want)


def test_golden_rng(ora, gold):
    for i, s in enumerate(gold["seeds"]):
        s = int(s)
        assert ora.splitmix64(s) == int(gold["splitmix64"][i])
        assert ora.mix_seed(s, 0x68617368) == int(gold["mix_seed_hash"][i])
        assert np.array_equal(ora.xorshift_stream(s, 16), gold["xorshift"][i])
        assert np.array_equal(ora.next_below_stream(s, 16, 64), gold["next_below16"][i])
        assert np.array_equal(ora.next_below_stream(s, P, 16), gold["next_below_p"][i])


def test_golden_make_config(ora, gold):
    for n, want in zip(gold["max_chain_n"], gold["max_chain"]):
        assert ora.default_max_chain(int(n)) == int(want)
    for (kind, n, b, t, seed), lf, row in zip(gold["make_config_params"], gold["make_config_lf"], gold["make_config_rows"]):
        c = ora.make_config(int(kind), int(n), float(lf), int(b), threshold=None if t < 0 else int(t), seed=int(seed))
        assert np.array_equal(row_from_cfg(c), row)


def test_golden_keygen(ora, gold):
    for s, want in zip(gold["keygen_seeds"], gold["keygen_keys"]):
        assert np.array_equal(ora.generate_keys(int(s), 256), want)
    for k, v in zip(gold["vfk_keys"], gold["vfk_values"]):
        assert ora.value_for_key(int(k)) == int(v)


def test_golden_sectors(ora, gold):
    cases = [("bcht", 16, 1.0), ("bcht", 16, 3.0), ("bcht", 32, 1.5), ("1cht", 1, 1.0), ("1cht", 1, 2.75),
             ("bp2ht", 8, 2.0), ("iht", 16, 1.48)]
    for (kind, b, pr), want in zip(cases, gold["sectors"]):
        assert ora.predict_sectors(kind, b, pr, "insert") == want[0]
        assert ora.predict_sectors(kind, b, pr, "find") == want[1]


def test_golden_tables(ora, gold):
    """Sequential builds are deterministic (same eviction stream), so the oracle must reproduce the reference's
    store BIT FOR BIT, and its find loop the same answers and probe counts."""
    for name in gold["table_cases"]:
        g = lambda f: gold[f"t_{name}_{f}"]  # noqa: E731
        cfg = cfg_from_row(g("cfg"))
        t = ora.table(cfg)
        r = t.build(g("keys"), g("values"))
        assert r["success"], name
        assert r["probes"] == int(g("insert_probes")), name
        assert np.array_equal(t.download_store(), g("store")), name
        q = np.concatenate([g("keys"), g("absent")])
        out, hits, probes = t.find_bulk(q)
        assert np.array_equal(out, g("find_out")), name
        assert probes == int(g("find_probes")), name
        ex = np.array([t.find_key_no_early_exit(int(k))[1] if t.find_key_no_early_exit(int(k))[0] else EMPTY for k in q[::5]],
                      dtype=np.uint32)
        assert np.array_equal(ex, g("find_exhaustive")[::5]), name
        # build() with value_for_key values
        t2 = ora.table(cfg)
        r2 = t2.build(g("keys"))
        assert r2["probes"] == int(g("build_probes")) and np.array_equal(t2.download_store(), g("build_store")), name


def test_golden_failed_build(ora, gold):
    cfg = cfg_from_row(gold["fail_cfg"])
    t = ora.table(cfg)
    r = t.build(gold["fail_keys"])
    assert not r["success"]
    assert r["inserted"] == int(gold["fail_inserted"])
    assert int(gold["fail_keys"][r["failed_index"]]) == int(gold["fail_key"])  # build stops at the first failed key
    assert np.array_equal(t.download_store(), gold["fail_store"])


# ---- 3. live against the compiled reference ------------------------------------------------------------------------------

@pytest.mark.parametrize("scenario,cfg_src", scenarios.ALL, ids=[s[0].__name__ for s in scenarios.ALL])
def test_scenarios_reference(ref, scenario, cfg_src):
    make = lambda cfg: scenarios.OracleAdapter(ref, cfg)  # noqa: E731
    src = ref.make_config if cfg_src == "make_config" else binding.craft
    scenario(make, src)


@pytest.mark.parametrize("kind,b,lf,t", [("bcht", 16, 0.9, None), ("bcht", 32, 0.97, None), ("1cht", 1, 0.85, None),
                                         ("bp2ht", 16, 0.8, None), ("iht", 16, 0.8, None), ("iht", 32, 0.9, 9),
                                         ("bcht", 64, 0.9, None), ("bcht", 2, 0.6, None)])
def test_oracle_equals_reference_live(ora, ref, kind, b, lf, t):
    n = 20_000
    keys = ref.generate_keys(1234 + b, 2 * n)
    assert np.array_equal(keys, ora.generate_keys(1234 + b, 2 * n))
    vals = np.arange(n, dtype=np.uint32) * np.uint32(2654435761)
    for attempt in range(30):
        cfg = ref.make_config(kind, n, lf, b, threshold=t, seed=ref.mix_seed(77, attempt))
        ocfg = ora.make_config(kind, n, lf, b, threshold=t, seed=ora.mix_seed(77, attempt))
        assert bytes(cfg) == bytes(ocfg)
        rt, ot = ref.table(cfg), ora.table(ocfg)
        rr = rt.insert_pairs(keys[:n], vals, stop_on_failure=False)
        orr = ot.insert_all(keys[:n], vals)
        assert rr["inserted"] == orr["inserted"] and rr["probes"] == orr["probes"]
        assert np.array_equal(rr["failed"], orr["failed"])
        assert np.array_equal(rt.download_store(), ot.download_store())
        if rr["success"]:
            break
    ro, rh, rp = rt.find_bulk(keys)
    oo, oh, op = ot.find_bulk(keys)
    assert np.array_equal(ro, oo) and rh == oh == n and rp == op
    assert rt.check_admissibility() == ot.check_admissibility() == 0
    # the reference's own checker (oracle.cpp:13-38) passes on the ORACLE-built layout (value_for_key values)
    o2 = ora.table(ocfg)
    if o2.build(keys[:n])["success"]:
        r2 = ref.table(cfg)
        r2.upload_store(o2.download_store())
        assert r2.check_membership(keys[:n], 1000, 5) == {"false_negatives": 0, "wrong_values": 0, "false_positives": 0}
