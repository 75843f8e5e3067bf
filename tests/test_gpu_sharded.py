"""The sharded table's device path on the one GPU this run has: a world of size 1 over NCCL exercises CudaShardOps
(K8 partition, K9 un-permute, local K4/K3) and the NCCL all_to_all_single plumbing end to end; with G = 1 every key is
owned by rank 0, and the answers must equal a plain single table's.  The N > 1 routing logic is covered on CPU by
tests/test_sharded_gloo.py."""
import socket

import numpy as np
import pytest

from conftest import random_values, unique_keys

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
EMPTY = 0xFFFFFFFF


@pytest.fixture(scope="module")
def nccl_world():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("exact", [None, False, True])  # None: a world of one needs no routing at all
@pytest.mark.parametrize("chunk", [1 << 26, 100_000])
def test_sharded_table_world_of_one(bht, nccl_world, chunk, exact):
    n = 700_000
    keys = unique_keys(n, 321, extra=n)
    vals = random_values(n, 321)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()  # noqa: E731
    cfg = bht.make_config("bcht", n, 0.9, 16, seed=12)
    st = bht.ShardedTable(cfg, device=0, chunk=chunk)
    o = st.insert(d(keys[:n]), d(vals), exact=exact)
    assert o.success and o.inserted == n and o.attempted == n
    assert st.inserted() == n
    q = np.concatenate([keys[:n:2], keys[n::2]])
    np.random.default_rng(0).shuffle(q)
    got = st.find(d(q), exact=exact).cpu().numpy().view(np.uint32)
    lookup = dict(zip(keys[:n].tolist(), vals.tolist()))
    want = np.array([lookup.get(int(x), EMPTY) for x in q], dtype=np.uint32)
    assert np.array_equal(got, want)
    # same answers as an unsharded table of the same configuration
    plain, o2 = bht.build(d(keys[:n]), cfg, d(vals), device=0)
    assert o2.success
    assert np.array_equal(plain.find(d(q)).cpu().numpy().view(np.uint32), want)


def test_sharded_build_in_chunks_takes_the_blocked_build(bht, nccl_world):
    """A shard that qualifies for the shared-memory-blocked build gets it however many chunks the keys arrive in
    (config 5 of BASELINE.json feeds 2^24-key chunks into 5e8-key shards): the received segments go through the chunked
    build (bht_build_begin / bht_build_feed_counted / bht_build_end), the store is written once, and the table equals
    the one a single bulk insert builds — same stored multiset, same probe totals for the finds."""
    n = 30_000_000  # 267 MB of slots: beyond the L2, so the default mode blocks
    keys, vals = bht.generate_unique_keys(3, 0, n, device=0)
    keys, vals = keys.view(torch.int32), vals.view(torch.int32)
    cfg = bht.make_config("bcht", n, 0.9, 16, seed=bht.mix_seed(1, 0x100))
    st = bht.ShardedTable(cfg, device=0, chunk=1 << 22)
    for exact in (False, None):  # the routed exchange (as N > 1 runs it), then the no-routing shortcut of a world of one
        st.ops.table.clear()
        launches0 = bht.kernel_launch_count()
        o = st.insert(keys, vals, exact=exact)
        assert o.success and o.inserted == n
        assert st.ops.table.last_build_schedule() == 3
        # 8 chunks: route (3 kernels) + one first-pass launch per chunk, then K10, K11, K4 once
        assert bht.kernel_launch_count() - launches0 <= 8 * 4 + 3 + 2
        out = st.find(keys, exact=exact)
        assert torch.equal(out, vals)
    plain = bht.HashTable(cfg, 0)
    assert plain.insert(keys, vals).success and plain.last_build_schedule() == 3
    _, fa = st.ops.table.find(keys, want_stats=True)
    _, fb = plain.find(keys, want_stats=True)
    assert fa.hits == fb.hits == n and abs(fa.probes - fb.probes) < 0.002 * fb.probes
    assert st.ops.table.occupied_slots() == n and st.ops.table.count_inadmissible() == 0


def test_fixed_segment_partition_against_numpy(bht):
    """bht_shard_partition_fixed: every key in the segment of its owner, counts on the device, padding untouched,
    the overflow flag raised (and nothing written out of bounds) when a segment is too small."""
    n, world = 1_000_003, 5
    keys = unique_keys(n, 77)
    vals = random_values(n, 77)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()  # noqa: E731
    cfg = bht.make_config("bcht", n, 0.9, 16, seed=5)
    ops = bht.CudaShardOps(cfg, 0)
    alpha, beta = bht.shard_constants(cfg.seed)
    lib = bht._lib.load()
    owner = np.array([lib.bht_shard_of_host(alpha, beta, world, int(k)) for k in keys[:20000]])
    cap = int(n / world * 1.05) & ~3
    # an element carries its value (inserts) or its position (finds): one call each
    sk, sv, _, counts = ops.partition_fixed(alpha, beta, world, d(keys), d(vals), False, cap)
    sk2, _, idx, counts2 = ops.partition_fixed(alpha, beta, world, d(keys), None, True, cap)
    torch.cuda.synchronize()
    assert int(ops.overflow.item()) == 0
    sk, sv, counts, sk2, idx, counts2 = (x.cpu().numpy() for x in (sk, sv, counts, sk2, idx, counts2))
    assert counts.sum() == n and np.array_equal(counts, counts2)
    lookup = dict(zip(keys.tolist(), vals.tolist()))
    for g in range(world):
        c = int(counts[g])
        seg_k = sk[g * cap:(g + 1) * cap].view(np.uint32)
        seg_v = sv[g * cap:g * cap + c].view(np.uint32)
        assert np.all(seg_k[c:] == EMPTY)  # padding: the sentinel key
        assert np.array_equal(np.array([lookup[int(k)] for k in seg_k[:3000]], dtype=np.uint32), seg_v[:3000])  # pairs stay pairs
        seg_k2 = sk2[g * cap:(g + 1) * cap].view(np.uint32)
        seg_i = idx[g * cap:(g + 1) * cap].view(np.uint32)
        assert np.all(seg_k2[c:] == EMPTY) and np.all(seg_i[c:] == EMPTY)  # padding: sentinel key, no index
        assert np.array_equal(keys[seg_i[:c]], seg_k2[:c])  # the index names the element's position in the input
        assert np.array_equal(np.sort(seg_k2[:c]), np.sort(seg_k[:c]))  # both calls route the same keys to g
        small = seg_i[:c][seg_i[:c] < 20000]
        assert np.all(owner[small] == g)
    with pytest.raises(ValueError):
        ops.partition_fixed(alpha, beta, world, d(keys), d(vals), True, cap)  # not both
    # a segment that is too small: flagged, counts clamped, neighbours' segments intact
    cap2 = int(n / world * 0.9) & ~3
    sk3, _, _, counts3 = ops.partition_fixed(alpha, beta, world, d(keys), None, False, cap2)
    torch.cuda.synchronize()
    assert int(ops.overflow.item()) == 1 and int(counts3.max().item()) == cap2
    sk3 = sk3.cpu().numpy().view(np.uint32)
    own3 = np.array([lib.bht_shard_of_host(alpha, beta, world, int(k)) for k in sk3[cap2:cap2 + 3000]])
    assert np.all(own3 == 1)
