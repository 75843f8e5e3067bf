"""Host-side logic of the sharded table on 2 ranks over gloo (CPU): counts exchange, (key, value) all-to-all, local
insert, reverse routing of answers, un-permute, result aggregation, chunk pipelining with ragged / empty ranks.

The device pieces (partition, probe kernels, un-permute) are replaced by a CPU stand-in built on the ORACLE, which
is allowed here because this is a test: the product's CudaShardOps has no CPU path."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EMPTY = 0xFFFFFFFF


class OracleShardOps:
    """CPU stand-in with the interface of paper_2108_07232_b200.sharded.CudaShardOps."""

    supports_counted = True
    cuckoo = True

    def __init__(self, cfg):
        from oracle import binding
        self.ora = binding.oracle()
        self.table_o = self.ora.table(binding.Config.from_buffer_copy(bytes(cfg)))
        self.table = self  # .table.inserted()
        self.overflow = torch.zeros(1, dtype=torch.int32)
        self.session = None
        self.host_reads = 0  # how often the routing logic pulled a count to the host (the exact exchange does, per chunk)

    def inserted(self):
        return self.table_o.inserted

    def empty(self, n):
        return torch.empty(n, dtype=torch.int32)

    def counts_tensor(self, counts):
        return torch.tensor(list(counts), dtype=torch.int64)

    def filled(self, n):
        return torch.full((n,), -1, dtype=torch.int32)

    def partition_fixed(self, alpha, beta, n_shards, keys, values, want_index, cap):
        k = keys.numpy().view(np.uint32)
        owner = np.array([self.ora.shard_of(alpha, beta, n_shards, int(x)) for x in k], dtype=np.int64)
        out_k, out_v, idx = self.filled(n_shards * cap), self.empty(n_shards * cap), self.filled(n_shards * cap)
        counts = torch.zeros(n_shards, dtype=torch.int64)
        for d in range(n_shards):
            at = np.flatnonzero(owner == d)
            if at.size > cap:
                self.overflow[0] = 1
                at = at[:cap]
            counts[d] = at.size
            out_k[d * cap:d * cap + at.size] = torch.from_numpy(k[at].view(np.int32).copy())
            if values is not None:
                out_v[d * cap:d * cap + at.size] = values[torch.from_numpy(at)]
            idx[d * cap:d * cap + at.size] = torch.from_numpy(at.astype(np.int32))
        return out_k, (out_v if values is not None else None), (idx if want_index else None), counts

    def build_begin(self, n_max):
        assert self.session is None
        self.session = [0, 0, 0, 0, None]

    def feed_counted(self, keys, values, cap, count):
        n = min(cap, int(count[0]))  # the stand-in reads the count; the product's kernels read it on the device
        o = self.insert(keys[:n], values[:n])
        ses = self.session
        ses[0] += o.attempted; ses[1] += o.inserted; ses[2] += o.failed; ses[3] += o.probes
        if ses[4] is None:
            ses[4] = o.failed_key

    def build_end(self):
        from paper_2108_07232_b200 import BuildOutcome
        a, i, f, p, fk = self.session
        self.session = None
        return BuildOutcome(f == 0, i, f, a, p, fk)

    def partition(self, alpha, beta, n_shards, keys, values, want_index):
        self.host_reads += 1
        k = keys.numpy().view(np.uint32)
        owner = np.array([self.ora.shard_of(alpha, beta, n_shards, int(x)) for x in k], dtype=np.int64)
        order = np.argsort(owner, kind="stable")
        counts = np.bincount(owner, minlength=n_shards).tolist()
        pk = torch.from_numpy(k[order].view(np.int32).copy())
        pv = torch.from_numpy(values.numpy()[order].copy()) if values is not None else None
        idx = torch.from_numpy(order.astype(np.int32)) if want_index else None
        return pk, pv, idx, counts

    def unpermute(self, answers, index, out):
        keep = index != -1  # padding slots of a fixed-segment exchange
        out[index[keep].long()] = answers[keep]

    def insert(self, keys, values):
        from paper_2108_07232_b200 import BuildOutcome
        k = keys.numpy().view(np.uint32)
        v = values.numpy().view(np.uint32)
        r = self.table_o.insert_all(k, v)
        failed = int(r["failed"].sum())
        fk = int(k[r["failed"]][0]) if failed else None
        return BuildOutcome(failed == 0, r["inserted"], failed, len(k), r["probes"], fk)

    def find(self, keys):
        k = keys.numpy().view(np.uint32)
        out = np.full(k.size, EMPTY, dtype=np.uint32)  # the sentinel key (padding) is answered EMPTY without a probe (find.cu)
        real = k != EMPTY
        out[real], _, _ = self.table_o.find_bulk(k[real])
        return torch.from_numpy(out.view(np.int32).copy())


def _worker(rank, world, port, n_per_rank, chunk, exact, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_07232_b200 as bht
        from conftest import random_values, unique_keys
        total = sum(n_per_rank)
        keys = unique_keys(total, 4242, extra=total)
        vals = random_values(total, 99)
        lo = sum(n_per_rank[:rank])
        hi = lo + n_per_rank[rank]
        cfg = bht.make_config("bcht", max(total // world, 1), 0.7, 16, seed=5)
        st = bht.ShardedTable(cfg, ops=OracleShardOps(cfg), chunk=chunk)
        mine_k = torch.from_numpy(keys[lo:hi].view(np.int32).copy())
        mine_v = torch.from_numpy(vals[lo:hi].view(np.int32).copy())
        outcome = st.insert(mine_k, mine_v, exact=exact)
        assert (st.ops.host_reads == 0) == (not exact)  # the fixed-segment exchange never pulls counts to the host
        assert outcome.success and outcome.inserted == total and outcome.attempted == total, outcome
        assert st.inserted() == total
        assert abs(st.realized_load() - total / (cfg.capacity * world)) < 1e-12
        # every key this shard holds is owned by this shard
        store = st.ops.table_o.download_store()
        held = (store[store != np.uint64(0xFFFFFFFFFFFFFFFF)] & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        lib = bht._lib.load()
        assert all(lib.bht_shard_of_host(st.alpha, st.beta, world, int(k)) == rank for k in held[:500])
        # queries: a different slice per rank, half present (inserted by ANY rank), half absent, shuffled
        rng = np.random.default_rng(rank)
        qn = n_per_rank[rank] + 17 * rank
        pres = rng.integers(0, total, size=qn // 2)
        absent = rng.integers(total, 2 * total, size=qn - qn // 2)
        pos = np.concatenate([pres, absent])
        rng.shuffle(pos)
        q_keys = keys[pos]
        want = np.where(pos < total, vals[np.minimum(pos, total - 1)], EMPTY).astype(np.uint32)
        reads0 = st.ops.host_reads
        got = st.find(torch.from_numpy(q_keys.view(np.int32).copy()), exact=exact).numpy().view(np.uint32)
        assert np.array_equal(got, want)
        assert (st.ops.host_reads == reads0) == (not exact)
        if not exact:
            # a segment too small for the chunk is reported, on every rank, not silently dropped
            st.segment_cap = lambda chunk_len: 8
            try:
                st.find(torch.from_numpy(q_keys.view(np.int32).copy()), exact=False)
                raise AssertionError("overflow went unnoticed")
            except bht.RoutingOverflow:
                pass
        # an insert that overfills reports failures consistently on all ranks
        q.put((rank, "ok", outcome.probes))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, "fail", traceback.format_exc() + str(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("n_per_rank,chunk", [([3000, 3000], 1 << 20), ([5000, 1200], 1024), ([0, 2500], 700)])
def test_sharded_table_two_ranks_gloo(n_per_rank, chunk, exact):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_per_rank, chunk, exact, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in results:
        assert status == "ok", f"rank {rank}: {info}"
    assert results[0][2] == results[1][2]  # aggregated probe count agrees on both ranks
