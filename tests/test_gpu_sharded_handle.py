"""The single-process sharded handle of the C ABI (bht_sharded_*, csrc/sharded.cu).  One GPU is
enough to run every step of it: device ids may repeat, so G shards on cuda:0 route, exchange (peer copies that are
plain device copies here), insert, find, send the answers back and un-permute exactly as G GPUs would."""
import numpy as np
import pytest

from conftest import random_values, unique_keys

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
EMPTY = 0xFFFFFFFF


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


def test_shard_constants_match_the_multi_process_router(bht):
    for seed in [0, 1, 7, 0xDEADBEEFCAFE, (1 << 64) - 1]:
        t_cfg = bht.make_config("bcht", 1000, 0.5, 16, seed=seed)
        local = bht.LocalShardedTable(t_cfg, [0])
        assert (local.alpha, local.beta) == tuple(bht.shard_constants(seed))
        local.close()


@pytest.mark.parametrize("kind,b,lf", [("bcht", 16, 0.85), ("1cht", 1, 0.6), ("bp2ht", 16, 0.7), ("iht", 16, 0.75)])
@pytest.mark.parametrize("shards", [1, 2, 5])
def test_sharded_handle_insert_find(bht, ora, kind, b, lf, shards):
    n_per = 60_001
    n = n_per * shards
    keys = unique_keys(n, 40 + shards, extra=5000)
    present, absent = keys[:n], keys[n:]
    values = random_values(n, 41)
    extra = {"threshold": 12} if kind == "iht" else {}
    # per-shard tables sized for their expected share plus the spread of the routing hash
    cfg = bht.make_config(kind, int(n_per * 1.05), lf, b, seed=77, **extra)
    table = bht.LocalShardedTable(cfg, [0] * shards)
    assert len(table) == shards
    # ragged slices: GPU g contributes a different number of pairs
    cuts = np.linspace(0, n, shards + 1).astype(np.int64)
    cuts[1:-1] += np.arange(1, shards) * 37
    k_slices = [dev(present[cuts[g]:cuts[g + 1]]) for g in range(shards)]
    v_slices = [dev(values[cuts[g]:cuts[g + 1]]) for g in range(shards)]
    o = table.insert(k_slices, v_slices)
    assert o.success and o.attempted == n and o.inserted == n and o.failed == 0
    # every pair lives in the shard the routing hash names, and only there
    owner = np.array([bht._lib.load().bht_shard_of_host(table.alpha, table.beta, shards, int(k)) for k in present[:2000]])
    total = 0
    for g in range(shards):
        shard = table.shard(g)
        assert shard.count_inadmissible() == 0
        got = host(shard.find(dev(present[:2000])))
        assert np.array_equal(got != EMPTY, owner == g)
        total += shard.occupied_slots()
        # the reference's checker accepts the shard's store
        otab = ora.table(__import__("conftest").to_oracle_cfg(cfg))
        otab.upload_store(shard.download_store())
        assert otab.check_admissibility() == 0
    assert total == n
    # queries come back in the caller's order, per slice; absent keys answer EMPTY
    q = np.concatenate([present, absent])
    want = np.concatenate([values, np.full(absent.size, EMPTY, dtype=np.uint32)])
    perm = np.random.Generator(np.random.MT19937(5)).permutation(q.size)
    q, want = q[perm], want[perm]
    qcuts = np.linspace(0, q.size, shards + 1).astype(np.int64)
    outs, stats = table.find([dev(q[qcuts[g]:qcuts[g + 1]]) for g in range(shards)], want_stats=True)
    for g in range(shards):
        assert np.array_equal(host(outs[g]), want[qcuts[g]:qcuts[g + 1]])
    assert stats.queries == q.size and stats.hits == n
    assert stats.value_sum == int(values.astype(np.uint64).sum())
    outs2 = table.find([dev(q[qcuts[g]:qcuts[g + 1]]) for g in range(shards)])
    for g in range(shards):
        assert np.array_equal(host(outs2[g]), want[qcuts[g]:qcuts[g + 1]])
    table.close()


def test_sharded_handle_keys_only_empty_slices_and_clear(bht, ora):
    shards, n = 3, 90_000
    keys = unique_keys(n, 91)
    cfg = bht.make_config("bcht", 40_000, 0.8, 16, seed=5)
    table = bht.LocalShardedTable(cfg, [0, 0, 0])
    slices = [dev(keys[:50_000]), None, dev(keys[50_000:])]  # GPU 1 contributes nothing
    o = table.insert(slices)                                  # values = value_for_key
    assert o.success and o.attempted == n
    want = ora.values_for_keys(keys)
    outs = table.find(slices)
    assert outs[1] is None
    assert np.array_equal(host(outs[0]), want[:50_000]) and np.array_equal(host(outs[2]), want[50_000:])
    table.clear()
    assert sum(table.shard(g).occupied_slots() for g in range(shards)) == 0
    outs = table.find(slices)
    assert np.all(host(outs[0]) == EMPTY) and np.all(host(outs[2]) == EMPTY)
    # the same keys into the same handle again, in two calls
    o1 = table.insert([dev(keys[:30_000]), dev(keys[30_000:45_000]), None])
    o2 = table.insert([None, None, dev(keys[45_000:])])
    assert o1.success and o2.success and o1.attempted + o2.attempted == n
    outs = table.find([dev(keys), None, None])
    assert np.array_equal(host(outs[0]), want)
    table.close()


def test_sharded_handle_reports_overfull_shards(bht):
    cfg = bht.make_config("bp2ht", 1000, 0.9, 8, seed=3)  # ~1100 slots per shard
    table = bht.LocalShardedTable(cfg, [0, 0])
    keys = unique_keys(2150, 8)
    o = table.insert([dev(keys[:1000]), dev(keys[1000:])])
    assert not o.success and o.attempted == 2150 and o.inserted + o.failed == 2150 and o.failed > 0 and o.failed_key is not None
    with pytest.raises(bht.CapacityError):
        table.insert([dev(unique_keys(4000, 9)), None])      # one shard would receive more than its capacity
    with pytest.raises(ValueError):
        table.insert([dev(keys[:10])])                        # one slice per shard
    table.close()
