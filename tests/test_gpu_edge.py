"""Edge cases of the CUDA path that the reference tests cover: empty and ragged inputs, the sentinel, error
behaviour, builds that fail, stability, single-bucket contention, store interchange, multi-call builds."""
import os

import numpy as np
import pytest

from conftest import ROOT, random_values, to_oracle_cfg, unique_keys

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
EMPTY = 0xFFFFFFFF


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


def packed(keys, values):
    return np.sort((values.astype(np.uint64) << np.uint64(32)) | keys.astype(np.uint64))


def stored(table):
    s = table.download_store()
    return np.sort(s[s != np.uint64(0xFFFFFFFFFFFFFFFF)])


def test_empty_and_ragged_sizes(bht):
    # test_table.cpp:208-216 (empty key set) and ragged tails around the warp / chunk sizes
    cfg = bht.make_config("bcht", 300_000, 0.8, 16, seed=2)
    table = bht.HashTable(cfg, 0)
    o = table.insert(np.empty(0, dtype=np.uint32), np.empty(0, dtype=np.uint32))
    assert o.success and o.inserted == 0 and o.probes == 0
    assert table.find(np.empty(0, dtype=np.uint32)).size == 0
    keys = unique_keys(250_000, 9)
    vals = random_values(250_000, 9)
    lo = 0
    for n in [1, 31, 32, 33, 255, 256, 257, 1023, 8191, 8193, 100_003]:
        o = table.insert(dev(keys[lo:lo + n]), dev(vals[lo:lo + n]))
        assert o.success and o.inserted == n and o.attempted == n
        lo += n
    assert table.inserted() == lo == table.occupied_slots()
    for n in [1, 31, 33, 257, 100_003, lo]:
        assert np.array_equal(host(table.find(dev(keys[:n]))), vals[:n])
        assert np.array_equal(table.find(keys[lo - n:lo]), vals[lo - n:lo])  # host path
    assert np.all(host(table.find(dev(keys[lo:lo + 5000]))) == EMPTY)
    table.clear()
    assert table.inserted() == 0 and table.occupied_slots() == 0
    assert np.all(host(table.find(dev(keys[:1000]))) == EMPTY)


def test_sentinel_query_and_duplicates_in_query(bht):
    cfg = bht.make_config("bcht", 1000, 0.5, 16, seed=3)
    table, o = bht.build(np.arange(1000, dtype=np.uint32), cfg, np.arange(1000, dtype=np.uint32) + 5, device=0)
    assert o.success
    q = np.array([EMPTY, 7, 7, 7, EMPTY, 999, 1000, 0], dtype=np.uint32)
    assert list(table.find(q)) == [EMPTY, 12, 12, 12, EMPTY, 1004, EMPTY, 5]


def test_error_behaviour(bht):
    cfg = bht.make_config("bcht", 16, 1.0, 16, seed=1)
    with pytest.raises(bht.CapacityError):  # table.cpp:225
        bht.build(np.arange(17, dtype=np.uint32), cfg, device=0)
    table = bht.HashTable(cfg, 0)
    bad = cfg.copy()
    bad.n_hashes = 2
    with pytest.raises(ValueError):  # table.cpp:22-23
        bht.HashTable(bad, 0)
    with pytest.raises(bht.KindMismatchError):  # require_kind, table.cpp:15-17
        table.insert(np.arange(4, dtype=np.uint32), np.arange(4, dtype=np.uint32), as_kind="bp2ht")
    with pytest.raises(bht.KindMismatchError):
        table.find(np.arange(4, dtype=np.uint32), as_kind="iht")
    with pytest.raises(bht.KindMismatchError):
        table.set_iht_prose_fallback(True)
    assert table.insert(np.arange(4, dtype=np.uint32), np.arange(4, dtype=np.uint32), as_kind="bcht").success
    one = bht.HashTable(bht.make_config("1cht", 100, 0.5, 1, seed=1), 0)
    assert one.insert(np.arange(4, dtype=np.uint32), np.arange(4, dtype=np.uint32), as_kind="bcht").success  # table.cpp:55
    with pytest.raises(ValueError):
        table.insert(dev(np.arange(4, dtype=np.uint32)), np.arange(4, dtype=np.uint32))  # mixed memory spaces
    with pytest.raises(ValueError):
        table.find(np.arange(4, dtype=np.float32))
    # a full table: further inserts fail like insert_pair does, they are not an error
    o = table.insert(np.arange(100, 116, dtype=np.uint32), np.arange(16, dtype=np.uint32))
    assert not o.success and o.failed >= 4 and o.inserted <= 12 and o.inserted + o.failed == 16


@pytest.mark.parametrize("kind,b,lf,t,max_chain", [("bp2ht", 8, 1.0, None, None), ("bp2ht", 16, 0.95, None, None),
                                                   ("iht", 16, 0.99, None, None), ("iht", 16, 0.97, 3, None),
                                                   ("bcht", 16, 0.999, None, 2), ("1cht", 1, 0.97, None, 6),
                                                   ("bcht", 4, 0.98, None, 1)])
def test_failed_builds_are_reported_consistently(bht, ora, kind, b, lf, t, max_chain):
    """Cells that do not build (SURVEY 'infeasible cells'): success=false, every dropped key is absent, every other key
    is found with its value, stored multiset == input minus dropped."""
    n = 80_000
    keys = unique_keys(n, 31 + b)
    vals = random_values(n, b)
    cfg = bht.make_config(kind, n, lf, b, threshold=t, seed=17, max_chain=max_chain)
    table, o = bht.build(dev(keys), cfg, dev(vals), device=0)
    assert not o.success and o.failed > 0 and o.inserted + o.failed == n and o.attempted == n
    dropped = table.failed_keys()
    assert dropped.size == o.failed and np.unique(dropped).size == dropped.size
    assert o.failed_key in set(dropped.tolist())
    assert np.isin(dropped, keys).all()
    got = host(table.find(dev(keys)))
    is_dropped = np.isin(keys, dropped)
    assert np.all(got[is_dropped] == EMPTY)
    assert np.array_equal(got[~is_dropped], vals[~is_dropped])
    assert np.array_equal(stored(table), packed(keys[~is_dropped], vals[~is_dropped]))
    assert table.inserted() == o.inserted == table.occupied_slots()
    assert table.count_inadmissible() == 0
    # the reference fails on the same cell (not necessarily on the same keys)
    ot = ora.table(to_oracle_cfg(cfg))
    assert not ot.build(keys, vals)["success"]
    # and agrees with the GPU about every query on the GPU-built layout
    ot.upload_store(table.download_store())
    want, _, _ = ot.find_bulk(keys)
    assert np.array_equal(got, want)


def test_single_bucket_contention_claims_exactly_b(bht):
    # acceptance.cpp:425-457 / test_bucket.cpp:79-95: many concurrent claimants, one bucket -> exactly b winners
    for kind, hashes in [("bp2ht", [(1, 0, 1), (1, 0, 1)]), ("iht", [(1, 0, 1)] * 3), ("bcht", [(1, 0, 1)] * 3)]:
        for b in [1, 2, 16, 64] if kind != "iht" else [2, 16, 64]:
            cfg = bht.craft_config(kind, 1, b, hashes, threshold=max(1, b // 2), max_chain=3)
            table = bht.HashTable(cfg, 0)
            n = 20_000
            keys = np.arange(1, n + 1, dtype=np.uint32)
            o = table.insert(dev(keys), dev(keys ^ np.uint32(0xABCD)))
            assert o.inserted == b and o.failed == n - b, (kind, b, o)
            s = table.download_store()
            k = (s & np.uint64(0xFFFFFFFF)).astype(np.uint32)
            v = (s >> np.uint64(32)).astype(np.uint32)
            assert np.unique(k).size == b and np.all(k != EMPTY)
            assert np.array_equal(v, k ^ np.uint32(0xABCD))  # no torn pairs (test_bucket.cpp:97-124)


@pytest.mark.parametrize("kind", ["bp2ht", "iht"])
def test_hot_buckets_in_a_wide_table_with_counter_claims(bht, kind):
    """Counter-claimed insert (csrc/insert_claim.cu): every key of a 600 k batch hashes to the same two (three) buckets of
    a 200 k-bucket table, so hundreds of thousands of lanes claim on the same counters at once.  Exactly the slots of those
    buckets are won, the counters' overshoot touches no neighbour, and a second batch into the same table places nothing."""
    nb, b, n = 200_000, 16, 600_000
    hashes = [(0, 4, nb), (0, 6, nb)] if kind == "bp2ht" else [(0, 4, nb), (0, 6, nb), (0, 9, nb)]
    cfg = bht.craft_config(kind, nb, b, hashes, threshold=12, max_chain=3)
    table = bht.HashTable(cfg, 0)
    table.set_blocked_insert(3)
    keys = np.arange(1, n + 1, dtype=np.uint32)
    o = table.insert(dev(keys), dev(keys ^ np.uint32(0x5A5A)))
    room = b * len(hashes)
    assert o.inserted == room and o.failed == n - room, o
    assert table.occupied_slots() == room
    s = table.download_store().reshape(nb, b)
    used = np.flatnonzero((s != np.uint64(0xFFFFFFFFFFFFFFFF)).any(axis=1))
    assert used.tolist() == sorted({h[1] for h in hashes})
    k = (s[used] & np.uint64(0xFFFFFFFF)).astype(np.uint32).ravel()
    v = (s[used] >> np.uint64(32)).astype(np.uint32).ravel()
    assert np.unique(k).size == room and np.array_equal(v, k ^ np.uint32(0x5A5A))
    o2 = table.insert(dev(keys + np.uint32(n)), dev(keys))
    assert o2.inserted == 0 and o2.failed == n and table.occupied_slots() == room
    # ordinary keys still land next to the hot buckets: a fresh uniform config on the same handle size
    cfg2 = bht.make_config(kind, 300_000, 0.8, b, seed=5)
    t2 = bht.HashTable(cfg2, 0)
    t2.set_blocked_insert(3)
    uk = unique_keys(300_000, 77)
    o3 = t2.insert(dev(uk), dev(uk))
    assert o3.success and np.array_equal(host(t2.find(dev(uk))), uk)


@pytest.mark.parametrize("kind,b,lf", [("bp2ht", 16, 0.8), ("iht", 16, 0.8), ("bp2ht", 32, 0.85)])
def test_stability_placed_pairs_never_move(bht, kind, b, lf):
    # test_table.cpp:262-284, acceptance.cpp:392-422
    n = 100_000
    keys = unique_keys(n, 55)
    vals = random_values(n, 55)
    table = bht.HashTable(bht.make_config(kind, n, lf, b, seed=8), 0)
    assert table.insert(dev(keys[:n // 2]), dev(vals[:n // 2])).success
    before = table.download_store()
    assert table.insert(dev(keys[n // 2:]), dev(vals[n // 2:])).success
    after = table.download_store()
    occupied = before != np.uint64(0xFFFFFFFFFFFFFFFF)
    assert np.array_equal(after[occupied], before[occupied])


def test_store_interchange_and_dump(bht, ora, tmp_path):
    n = 30_000
    keys = unique_keys(n, 66)
    cfg = bht.make_config("iht", n, 0.8, 16, seed=4)
    table, o = bht.build(dev(keys), cfg, device=0)
    assert o.success
    path = tmp_path / "store.bin"
    table.dump_store(str(path))  # table.cpp:41-51: LE u64 per slot, bucket order
    raw = np.fromfile(path, dtype="<u8")
    assert np.array_equal(raw, table.download_store())
    with pytest.raises(OSError):
        table.dump_store(str(tmp_path / "no_such_dir" / "x.bin"))
    # slot_at / poke_slot (table.hpp:53-56): corrupt one value, the oracle's checker sees exactly one wrong value
    ot = ora.table(to_oracle_cfg(cfg))
    idx = int(np.nonzero(raw != np.uint64(0xFFFFFFFFFFFFFFFF))[0][5])
    slot = table.slot_at(idx)
    assert slot == int(raw[idx])
    k = slot & 0xFFFFFFFF
    table.poke_slot(idx, bht.pack_pair(k, 12345))
    assert host(table.find(dev(np.array([k], dtype=np.uint32))))[0] == 12345
    ot.upload_store(table.download_store())
    want, _, _ = ot.find_bulk(keys)
    assert int((want != ora.values_for_keys(keys)).sum()) == 1  # test_oracle.cpp:29-46 shape
    # a foreign key poked into a bucket it does not hash to is an admissibility violation (test_oracle.cpp:48-64)
    empty_idx = int(np.nonzero(raw == np.uint64(0xFFFFFFFFFFFFFFFF))[0][0])
    foreign = next(x for x in range(1, 1000) if all(table.bucket_of(i, x) != empty_idx // 16 for i in range(3)))
    table.poke_slot(empty_idx, bht.pack_pair(foreign, 1))
    assert table.count_inadmissible() == 1


def test_multi_stream_concurrent_finds(bht):
    n = 400_000
    keys = unique_keys(n, 88)
    vals = random_values(n, 88)
    table, o = bht.build(dev(keys), bht.make_config("bcht", n, 0.9, 16, seed=6), dev(vals), device=0)
    assert o.success
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    dk = dev(keys)
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            outs.append(table.find(dk[i::4].contiguous(), stream=s))
    torch.cuda.synchronize()
    for i, o_ in enumerate(outs):
        assert np.array_equal(host(o_), vals[i::4])


def test_device_key_generator_and_shard_routing(bht):
    from paper_2108_07232_b200 import _lib
    lib = _lib.load()
    seed = 0x1234ABCD5678
    k, v = bht.generate_unique_keys(seed, 1000, 1 << 20, device=0)
    k, v = host(k), host(v)
    assert np.unique(k).size == k.size and not np.any(k == EMPTY) and not np.any(v == EMPTY)
    assert [int(x) for x in k[:50]] == [lib.bht_unique_key_host(seed, 1000 + i) for i in range(50)]
    assert [int(x) for x in v[:50]] == [lib.bht_synthetic_value_host(seed, int(x)) for x in k[:50]]
    with pytest.raises(ValueError):
        bht.generate_unique_keys(seed, 0xFFFFFFF0, 100, device=0)
    # K8 partition + K9 un-permute against numpy
    a, b = bht.shard_constants(5)
    ops = bht.CudaShardOps(bht.make_config("bcht", 1000, 0.5, 16, seed=1), 0)
    for n_shards in [1, 2, 8, 7]:
        dk, dv = dev(k), dev(v)
        pk, pv, idx, counts = ops.partition(a, b, n_shards, dk, dv, True)
        owner = np.array([lib.bht_shard_of_host(a, b, n_shards, int(x)) for x in k[:2000]])
        pk, pv, idx = host(pk), host(pv), host(idx).astype(np.int64)
        assert sum(counts) == k.size
        assert np.array_equal(k[idx], pk) and np.array_equal(v[idx], pv)  # routed element i came from position idx[i]
        assert np.unique(idx).size == k.size
        bounds = np.cumsum([0] + counts)
        full_owner = ((((a * k.astype(object) + b) % 4294967291) * n_shards) >> 32).astype(np.int64) if k.size <= 4096 else None
        for s in range(n_shards):
            seg = pk[bounds[s]:bounds[s + 1]]
            sample = seg[:: max(1, seg.size // 200)]
            assert all(lib.bht_shard_of_host(a, b, n_shards, int(x)) == s for x in sample)
        assert np.array_equal(np.bincount(owner, minlength=n_shards)[:n_shards] > 0, np.array(counts) > 0) or n_shards > 2
        out = torch.empty(k.size, dtype=torch.int32, device="cuda")
        ops.unpermute(dev(pv), dev(idx.astype(np.uint32)), out)
        assert np.array_equal(host(out), v)


@pytest.mark.parametrize("b,skew_regions", [(16, 2), (8, 1), (32, 3)])
def test_blocked_build_with_skewed_first_buckets(bht, ora, b, skew_regions):
    """The shared-memory-blocked build sizes its group segments, bins and stash for a uniform hash (mean + 6 sigma).  A key
    set whose first buckets crowd into a few regions overflows all three; the surplus must take the spill list and the
    general kernel, and the table must still hold exactly the inserted set (csrc/build_blocked.cu)."""
    n = 150_001
    cfg = bht.make_config("bcht", n, 0.85, b, seed=bht.mix_seed(41, b))
    region_buckets = (64 * 1024) // (8 * b)
    pool = unique_keys(6 * n, 500 + b)
    h0 = host(bht.hash_keys(int(cfg.alpha[0]), int(cfg.beta[0]), int(cfg.range[0]), dev(pool)))
    crowded = pool[h0 < skew_regions * region_buckets]
    spread = pool[h0 >= skew_regions * region_buckets]
    k_crowded = min(crowded.size, int(0.85 * skew_regions * region_buckets * b * 1.5))  # 1.5x what those regions can hold
    keys = np.concatenate([crowded[:k_crowded], spread[:n - k_crowded]])
    np.random.Generator(np.random.MT19937(7)).shuffle(keys)
    values = random_values(n, 9 * b)
    table = bht.HashTable(cfg, 0)
    table.set_blocked_insert(3)
    o = table.insert(dev(keys), dev(values))
    assert o.attempted == n and o.inserted + o.failed == n
    assert table.occupied_slots() == o.inserted and table.count_inadmissible() == 0
    got = host(table.find(dev(keys)))
    if o.success:
        assert np.array_equal(got, values)
        assert np.array_equal(stored(table), packed(keys, values))
        otab = ora.table(to_oracle_cfg(cfg))
        otab.upload_store(table.download_store())
        assert otab.check_admissibility() == 0
        want, hits, probes = otab.find_bulk(keys)
        assert hits == n and np.array_equal(want, values)
    else:  # dropped pairs are reported and are exactly the ones that are not found
        dropped = table.failed_keys()
        assert dropped.size == o.failed
        missing = keys[got == EMPTY]
        assert np.array_equal(np.sort(missing), np.sort(dropped))
    # the same key set into a NON-empty table (region_build loads the regions, finds the loads, claims after them)
    table2 = bht.HashTable(cfg, 0)
    table2.set_blocked_insert(3)
    half = n // 2
    o1 = table2.insert(dev(keys[:half]), dev(values[:half]))
    o2 = table2.insert(dev(keys[half:]), dev(values[half:]))
    assert table2.occupied_slots() == o1.inserted + o2.inserted and table2.count_inadmissible() == 0
    if o1.success and o2.success:
        assert np.array_equal(host(table2.find(dev(keys))), values)


@pytest.mark.parametrize("mode", [0, 3])
def test_deferred_clear_is_indistinguishable_from_a_fill(bht, mode):
    """bht_create / bht_clear defer the fill of the store (csrc/capi.cu, clear_pending): a shared-memory-blocked build into
    the empty table writes every region once, empty slots included, and every other use fills first.  Whatever follows a
    clear must see an empty table, and nothing of the previous contents may survive a clear + build."""
    n = 150_001
    a, b_keys = unique_keys(2 * n, 321)[:n], unique_keys(2 * n, 321)[n:]
    cfg = bht.make_config("bcht", n, 0.85, 16, seed=4)
    table = bht.HashTable(cfg, 0)                       # created, never filled yet
    assert table.occupied_slots() == 0
    table = bht.HashTable(cfg, 0)
    assert np.all(host(table.find(dev(a[:1000]))) == EMPTY)
    table = bht.HashTable(cfg, 0)
    assert np.all(table.download_store() == np.uint64(0xFFFFFFFFFFFFFFFF))
    table = bht.HashTable(cfg, 0)
    table.set_blocked_insert(mode)
    assert table.insert(dev(a), dev(a)).success
    assert np.array_equal(host(table.find(dev(a))), a)
    table.clear()
    assert table.inserted() == 0
    assert np.all(host(table.find(dev(a))) == EMPTY)    # find after a deferred clear
    assert table.insert(dev(a), dev(a)).success
    table.clear()
    m = n // 3
    assert table.insert(dev(b_keys[:m]), dev(b_keys[:m])).success   # clear + build: the build writes the whole store
    assert table.occupied_slots() == m and table.count_inadmissible() == 0
    assert np.all(host(table.find(dev(a))) == EMPTY)
    assert np.array_equal(host(table.find(dev(b_keys[:m]))), b_keys[:m])
    table.clear()
    table.clear()
    assert table.occupied_slots() == 0
    assert int((table.device_store() != -1).sum().item()) == 0   # the zero-copy view is filled before it is handed out
    # a small (unblocked) batch right after a clear
    assert table.insert(dev(a[:100]), dev(a[:100])).success
    assert table.occupied_slots() == 100 and np.array_equal(host(table.find(dev(a[:100]))), a[:100])
