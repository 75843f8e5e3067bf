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


@pytest.mark.parametrize("chunk", [1 << 26, 100_000])
def test_sharded_table_world_of_one(bht, nccl_world, chunk):
    n = 700_000
    keys = unique_keys(n, 321, extra=n)
    vals = random_values(n, 321)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()  # noqa: E731
    cfg = bht.make_config("bcht", n, 0.9, 16, seed=12)
    st = bht.ShardedTable(cfg, device=0, chunk=chunk)
    o = st.insert(d(keys[:n]), d(vals))
    assert o.success and o.inserted == n and o.attempted == n
    assert st.inserted() == n
    q = np.concatenate([keys[:n:2], keys[n::2]])
    np.random.default_rng(0).shuffle(q)
    got = st.find(d(q)).cpu().numpy().view(np.uint32)
    lookup = dict(zip(keys[:n].tolist(), vals.tolist()))
    want = np.array([lookup.get(int(x), EMPTY) for x in q], dtype=np.uint32)
    assert np.array_equal(got, want)
    # same answers as an unsharded table of the same configuration
    plain, o2 = bht.build(d(keys[:n]), cfg, d(vals), device=0)
    assert o2.success
    assert np.array_equal(plain.find(d(q)).cpu().numpy().view(np.uint32), want)
