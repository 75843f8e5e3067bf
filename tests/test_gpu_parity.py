"""GPU parity tests proper: the CUDA path, called through the C ABI, against the CPU oracle on the same inputs.

Bar: bit-exact. For every query the found / not-found flag and the value equal the oracle's; the stored
(key, value) multiset equals the inserted set; every stored pair is admissible.  Slot layout may differ from a
sequential CPU build (concurrent insertion order), so stores are never compared positionally.
"""
import numpy as np
import pytest

from conftest import random_values, to_oracle_cfg, unique_keys

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EMPTY = 0xFFFFFFFF


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


def stored_pairs(store):
    s = store[store != np.uint64(0xFFFFFFFFFFFFFFFF)]
    return np.sort(s)


def packed(keys, values):
    return np.sort((values.astype(np.uint64) << np.uint64(32)) | keys.astype(np.uint64))


CASES = [
    # kind, b, lf, threshold
    ("bcht", 16, 0.9, None),
    ("bcht", 16, 0.99, None),
    ("bcht", 8, 0.9, None),
    ("bcht", 32, 0.9, None),
    ("bcht", 1, 0.5, None),
    ("bcht", 2, 0.7, None),
    ("bcht", 4, 0.8, None),
    ("bcht", 64, 0.9, None),
    ("1cht", 1, 0.8, None),
    ("1cht", 1, 0.9, None),
    ("bp2ht", 16, 0.8, None),
    ("bp2ht", 32, 0.9, None),
    ("bp2ht", 8, 0.6, None),
    ("iht", 16, 0.8, None),
    ("iht", 16, 0.86, 6),
    ("iht", 32, 0.9, None),
    ("iht", 8, 0.6, None),
]


# ---- hash stage (hash.hpp:21-23) -------------------------------------------------------------------------------

def test_hash_stage_known_answers(bht):
    # proj/tests/test_hash.cpp:14-28
    for (a, b, r, k, want) in [(1, 0, 10, 7, 7), (3, 4, 3, 7, 1), (2, 0, 5, 4294967290, 4)]:
        got = host(bht.hash_keys(a, b, r, dev(np.array([k], dtype=np.uint32))))
        assert int(got[0]) == want


def test_hash_stage_random_parity(bht, ora):
    rng = np.random.Generator(np.random.MT19937(3))
    keys = rng.integers(0, 1 << 32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    keys[:4] = [0, 1, 0xFFFFFFFE, 0xFFFFFFFF]
    p = 4294967291
    for (a, b, r) in [(p - 1, p - 1, 62_500_000), (1, 0, 1), (p - 1, 0, (1 << 32) - 1), (3191871890, 3460072972, 3472223),
                      (12345, 678, 2), (2654435761, 40503, 1 << 31)]:
        got = host(bht.hash_keys(a, b, r, dev(keys)))
        want = ora.bucket_index_many(a, b, r, keys)
        assert np.array_equal(got.astype(np.uint64), want.astype(np.uint64)), (a, b, r)


# ---- bulk find on a table built by the CPU oracle ----------------------------------------------------------------

@pytest.mark.parametrize("kind,b,lf,t", CASES)
def test_find_on_oracle_built_table(bht, ora, kind, b, lf, t):
    n = 60_000
    keys = unique_keys(n, 100 + b, extra=n)
    present, absent = keys[:n], keys[n:]
    values = random_values(n, b)
    for attempt in range(20):  # fresh hash constants per failed build, as run_trial does (experiments.cpp:69-82)
        cfg = bht.make_config(kind, n, lf, b, threshold=t, seed=bht.mix_seed(5, 0x100 + attempt))
        otab = ora.table(to_oracle_cfg(cfg))
        if otab.build(present, values)["success"]:
            break
    else:
        pytest.skip("configuration does not build in the oracle either")
    table = bht.HashTable(cfg, 0)
    table.upload_store(otab.download_store())
    assert table.inserted() == n
    assert table.occupied_slots() == otab.occupied_slots() == n
    assert table.count_inadmissible() == 0
    queries = np.concatenate([present, absent])
    np.random.default_rng(1).shuffle(queries)
    got, stats = table.find(dev(queries), want_stats=True)
    want, hits, probes = otab.find_bulk(queries)
    assert np.array_equal(host(got), want)
    assert stats.hits == hits == n
    assert stats.probes == probes  # one probe per bucket read: identical accounting (probe_stats.hpp)
    assert stats.value_sum == int(want[want != EMPTY].astype(np.uint64).sum())
    # exhaustive find (oracle.cpp:56-63) agrees with the early-exit find
    got2 = table.find_exhaustive(dev(queries))
    assert np.array_equal(host(got2), want)


# ---- bulk insert: GPU build checked by the CPU oracle -------------------------------------------------------------

@pytest.mark.parametrize("kind,b,lf,t", CASES)
def test_build_parity(bht, ora, kind, b, lf, t):
    n = 60_000
    keys = unique_keys(n, 200 + b, extra=n)
    present, absent = keys[:n], keys[n:]
    values = random_values(n, 7 * b)
    for attempt in range(20):
        cfg = bht.make_config(kind, n, lf, b, threshold=t, seed=bht.mix_seed(9, 0x100 + attempt))
        table, outcome = bht.build(dev(present), cfg, dev(values), device=0)
        if outcome.success:
            break
        table.close()
    else:
        pytest.skip("configuration does not build")
    assert outcome.inserted == n and outcome.failed == 0 and outcome.failed_key is None
    assert table.inserted() == n and table.occupied_slots() == n
    assert abs(table.realized_load() - n / cfg.capacity) < 1e-12
    assert table.count_inadmissible() == 0
    store = table.download_store()
    # stored multiset == inserted set
    assert np.array_equal(stored_pairs(store), packed(present, values))
    # the CPU oracle, reading the GPU-built layout, passes its own checks and answers like the GPU
    otab = ora.table(to_oracle_cfg(cfg))
    otab.upload_store(store)
    assert otab.check_admissibility() == 0
    queries = np.concatenate([present, absent])
    want, hits, probes = otab.find_bulk(queries)
    assert hits == n
    assert np.array_equal(want[:n], values) and np.all(want[n:] == EMPTY)
    got, stats = table.find(dev(queries), want_stats=True)
    assert np.array_equal(host(got), want)
    assert stats.probes == probes
    # an independent sequential oracle build of the same pairs gives the same answers
    o2 = ora.table(to_oracle_cfg(cfg))
    if o2.build(present, values)["success"]:
        want2, _, _ = o2.find_bulk(queries)
        assert np.array_equal(host(got), want2)


@pytest.mark.parametrize("mode", [2, 3])
@pytest.mark.parametrize("kind,b,lf,t", CASES)
def test_build_parity_routed(bht, ora, monkeypatch, kind, b, lf, t, mode):
    """The blocked builds — mode 2: pairs routed by the L2-sized table region of their first bucket (packed-pair input
    of the insert kernels); mode 3: pairs binned by shared-memory-sized region, regions built in shared memory, the
    rest through the general kernel — give the same stored multiset, admissible, same answers as a sequential oracle
    build of the same pairs."""
    n = 150_001  # not a multiple of the router's group / tile sizes
    keys = unique_keys(n, 300 + b, extra=n)
    present, absent = keys[:n], keys[n:]
    values = random_values(n, 11 * b)
    monkeypatch.setenv("BHT_REGION_MB", "1")
    bht.reload_tuning()  # the knobs are read once per process
    for attempt in range(20):
        cfg = bht.make_config(kind, n, lf, b, threshold=t, seed=bht.mix_seed(13, 0x100 + attempt))
        table = bht.HashTable(cfg, 0)
        table.set_blocked_insert(mode)  # whatever the sizes (auto mode only blocks multi-million-key batches)
        table.set_tail_throttle(lf >= 0.99)  # the throttled second launch for the pairs beyond load 0.98
        outcome = table.insert(dev(present), dev(values))
        if outcome.success:
            break
        table.close()
    else:
        pytest.skip("configuration does not build")
    assert outcome.inserted == n and outcome.failed == 0
    assert table.inserted() == n and table.occupied_slots() == n
    assert table.count_inadmissible() == 0
    store = table.download_store()
    assert np.array_equal(stored_pairs(store), packed(present, values))
    otab = ora.table(to_oracle_cfg(cfg))
    otab.upload_store(store)
    assert otab.check_admissibility() == 0
    queries = np.concatenate([present, absent])
    want, hits, probes = otab.find_bulk(queries)
    assert hits == n and np.array_equal(want[:n], values) and np.all(want[n:] == EMPTY)
    got, stats = table.find(dev(queries), want_stats=True)
    assert np.array_equal(host(got), want) and stats.probes == probes
    # a second routed batch into the non-empty table (unaligned device slices: the router's element-load path)
    if kind in ("bcht", "1cht") and lf <= 0.9:
        extra = absent[1:2001]
        ev = random_values(2000, 5)
        o2 = table.insert(dev(np.concatenate([[0], extra]))[1:], dev(np.concatenate([[0], ev]))[1:])
        if o2.success:
            got2 = host(table.find(dev(extra)))
            assert np.array_equal(got2, ev)
            assert table.occupied_slots() == n + 2000 and table.count_inadmissible() == 0


@pytest.mark.parametrize("kind,b,lf,mode", [("bcht", 16, 0.9, 3), ("bcht", 16, 0.9, 2), ("bcht", 8, 0.85, 0), ("1cht", 1, 0.7, 1),
                                            ("bp2ht", 16, 0.75, 3), ("bp2ht", 16, 0.75, 0), ("iht", 16, 0.8, 3), ("iht", 32, 0.8, 0)])
@pytest.mark.parametrize("space", ["device", "host"])
def test_keys_only_insert_pairs_every_key_with_value_for_key(bht, ora, kind, b, lf, mode, space):
    """values = NULL through the C ABI: build(keys, cfg) pairs key k with value_for_key(k) (table.cpp:234, keygen.hpp:23-26).
    Same stored multiset and answers as the explicit-values call, for every schedule, from device and from host memory,
    in one batch and in ragged batches (and with the throttled tail, which reads the derived array at an offset)."""
    n = 180_001
    keys = unique_keys(n, 900 + b)
    keys[5] = np.uint32(0xFFFFFFFF ^ 0x5A5A5A5A)  # the one key whose image would be the sentinel (keygen.hpp:25)
    keys = np.unique(keys)
    np.random.Generator(np.random.MT19937(3)).shuffle(keys)
    n = keys.size
    want_vals = ora.values_for_keys(keys)
    assert want_vals[np.flatnonzero(keys == np.uint32(0xFFFFFFFF ^ 0x5A5A5A5A))[0]] == np.uint32(0x7FFFFFFF)
    extra = {"threshold": int(0.8 * b)} if kind == "iht" else {}
    cfg = bht.make_config(kind, n, lf, b, seed=bht.mix_seed(5, b), **extra)
    src = dev(keys) if space == "device" else keys
    for cuts, throttle in [((0, n), False), ((0, 1, 70_003, n), True)]:
        table = bht.HashTable(cfg, 0)
        table.set_blocked_insert(mode)
        table.set_tail_throttle(throttle)
        ok = True
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            ok &= table.insert(src[lo:hi]).success
        assert ok and table.occupied_slots() == n and table.count_inadmissible() == 0
        assert np.array_equal(stored_pairs(table.download_store()), packed(keys, want_vals))
        assert np.array_equal(host(table.find(dev(keys))), want_vals)
        table.close()


def test_build_default_values_and_host_memory(bht, ora):
    """values=None -> value_for_key (table.cpp:234); host arrays go through the staged PCIe path."""
    n = 300_000
    keys = unique_keys(n, 77, extra=1000)
    present, absent = keys[:n], keys[n:]
    cfg = bht.make_config("bcht", n, 0.9, 16, seed=3)
    table, outcome = bht.build(present, cfg, device=0)  # numpy (host) input
    assert outcome.success
    q = np.concatenate([present, absent])
    got = table.find(q)  # host in, host out
    assert isinstance(got, np.ndarray)
    want = ora.values_for_keys(q)
    want[n:] = EMPTY
    assert np.array_equal(got, want)
    got_dev = host(table.find(dev(q)))
    assert np.array_equal(got_dev, want)
