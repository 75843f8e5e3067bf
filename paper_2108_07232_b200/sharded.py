"""Sharded table: the key space range-partitioned across the GPUs of one box, one process per GPU.

No reference counterpart (the reference is single-process).  Ownership is a function of
the key alone, ``owner(k) = (g(k) * G) >> 32`` with ``g(k) = (a*k + b) mod p`` an independent member of the
table's hash family (hash.hpp:21-23), so all candidate buckets of a key live in one shard and every shard
is an ordinary single-GPU table.

    insert:  partition (device) -> counts all-to-all -> (key, value) all-to-all -> local bulk insert
    find:    partition (device) -> counts all-to-all -> key all-to-all -> local bulk find
             -> answers all-to-all back -> un-permute into query order (device)

The exchange runs on ``torch.distributed`` (NCCL over NVLink on GPUs).  Work is cut into chunks and the
all-to-all of chunk i+1 is issued asynchronously before the probe kernel of chunk i, so routing hides under
the HBM-bound probe work.  The per-rank pieces (partition, probe, un-permute) are behind a small ``ops``
object: ``CudaShardOps`` is the product implementation (C ABI kernels); tests inject a CPU stand-in to run the
routing logic on ``gloo``.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .table import BuildOutcome, HashTable, _check, _stream_ptr, mix_seed

_P = _lib.HASH_PRIME
_M64 = (1 << 64) - 1


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def shard_constants(seed: int):
    """(alpha, beta) of the routing hash, drawn as draw_hash_params does (keygen.cpp:14-26) from the stream
    xorshift_rng(mix_seed(seed, 'shar')) so that it is independent of the table's own constants."""
    state = _splitmix64(mix_seed(seed, 0x73686172)) or 0xD1B54A32D192ED03

    def next_below(bound):
        nonlocal state
        x = state
        x ^= (x << 13) & _M64
        x ^= x >> 7
        x ^= (x << 17) & _M64
        state = x
        return ((x >> 32) * bound) >> 32

    alpha = 1 + next_below(_P - 1)
    beta = next_below(_P)
    return alpha, beta


class CudaShardOps:
    """Per-rank device work of the sharded table, all through the C ABI."""

    def __init__(self, cfg, device: int):
        self.device = int(device)
        self.table = HashTable(cfg, self.device)
        self._lib = _lib.load()

    @property
    def torch_device(self):
        return torch.device("cuda", self.device)

    def empty(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=torch.int32, device=self.torch_device)

    def partition(self, alpha: int, beta: int, n_shards: int, keys: torch.Tensor, values: Optional[torch.Tensor],
                  want_index: bool):
        n = keys.numel()
        out_keys = self.empty(n)
        out_vals = self.empty(n) if values is not None else None
        index = self.empty(n) if want_index else None
        counts = (C.c_uint64 * n_shards)()
        _check(self._lib.bht_shard_partition(
            alpha, beta, n_shards, keys.data_ptr(), values.data_ptr() if values is not None else None, n,
            out_keys.data_ptr(), out_vals.data_ptr() if out_vals is not None else None,
            index.data_ptr() if index is not None else None, counts, self.device,
            _stream_ptr(None, self.device)))
        return out_keys, out_vals, index, [int(c) for c in counts]

    def unpermute(self, answers: torch.Tensor, index: torch.Tensor, out: torch.Tensor) -> None:
        _check(self._lib.bht_shard_unpermute(answers.data_ptr(), index.data_ptr(), answers.numel(), out.data_ptr(),
                                             self.device, _stream_ptr(None, self.device)))

    def insert(self, keys: torch.Tensor, values: torch.Tensor) -> BuildOutcome:
        return self.table.insert(keys, values)

    def find(self, keys: torch.Tensor) -> torch.Tensor:
        out = self.empty(keys.numel())
        self.table.find(keys, out)
        return out

    def counts_tensor(self, counts: Sequence[int]) -> torch.Tensor:
        return torch.tensor(list(counts), dtype=torch.int64, device=self.torch_device)


class ShardedTable:
    """One logical table over ``world_size`` shards; call every method collectively on all ranks."""

    def __init__(self, cfg_per_shard, group=None, ops=None, device: Optional[int] = None, chunk: int = 1 << 26,
                 route_seed: Optional[int] = None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if ops is None:
            ops = CudaShardOps(cfg_per_shard, torch.cuda.current_device() if device is None else device)
        self.ops = ops
        self.cfg = cfg_per_shard
        self.chunk = int(chunk)
        self.alpha, self.beta = shard_constants(cfg_per_shard.seed if route_seed is None else route_seed)

    # -- routing pieces
    def _exchange_counts(self, send_counts: List[int]) -> List[int]:
        send = self.ops.counts_tensor(send_counts)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        return [int(c) for c in recv.tolist()]

    def _all_to_all(self, send: torch.Tensor, send_counts: List[int], recv_counts: List[int], async_op: bool):
        recv = self.ops.empty(sum(recv_counts))
        work = dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=send_counts,
                                      group=self.group, async_op=async_op)
        return recv, work

    def _chunks(self, n: int):
        # every rank must issue the same number of collectives: agree on the max chunk count
        mine = max(1, -(-n // self.chunk))
        t = self.ops.counts_tensor([mine])
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        total = int(t.item())
        for c in range(total):
            lo = min(c * self.chunk, n)
            yield lo, min(lo + self.chunk, n)

    @staticmethod
    def _i32(x: torch.Tensor) -> torch.Tensor:
        return x.view(torch.int32) if x.dtype == torch.uint32 else x

    # -- the hot path
    def insert(self, keys: torch.Tensor, values: torch.Tensor) -> BuildOutcome:
        """Routes this rank's (key, value) pairs to their owners and bulk-inserts what this rank owns.
        Returns the outcome aggregated over all ranks."""
        keys, values = self._i32(keys), self._i32(values)
        totals = [0, 0, 0, 0]  # attempted, inserted, failed, probes
        failed_key = None
        pending = None

        def drain(p):
            nonlocal failed_key
            rk, rv, wk, wv = p
            if wk is not None:
                wk.wait()
                wv.wait()
            o = self.ops.insert(rk, rv)
            totals[0] += o.attempted
            totals[1] += o.inserted
            totals[2] += o.failed
            totals[3] += o.probes
            if o.failed_key is not None and failed_key is None:
                failed_key = o.failed_key

        for lo, hi in self._chunks(keys.numel()):
            pk, pv, _, send_counts = self.ops.partition(self.alpha, self.beta, self.world, keys[lo:hi], values[lo:hi],
                                                        False)
            recv_counts = self._exchange_counts(send_counts)
            rk, wk = self._all_to_all(pk, send_counts, recv_counts, True)
            rv, wv = self._all_to_all(pv, send_counts, recv_counts, True)
            if pending is not None:
                drain(pending)  # probe kernels of the previous chunk run under this chunk's exchange
            pending = (rk, rv, wk, wv)
        if pending is not None:
            drain(pending)

        t = self.ops.counts_tensor(totals + [-1 if failed_key is None else failed_key])
        agg = t[:4].clone()
        dist.all_reduce(agg, op=dist.ReduceOp.SUM, group=self.group)
        fk = t[4:].clone()
        dist.all_reduce(fk, op=dist.ReduceOp.MAX, group=self.group)
        attempted, inserted, failed, probes = (int(x) for x in agg.tolist())
        fkv = int(fk.item())
        return BuildOutcome(inserted == attempted, inserted, failed, attempted, probes, None if fkv < 0 else fkv)

    def find(self, keys: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Answers this rank's queries in the caller's order: out[i] = value or EMPTY_VALUE."""
        keys = self._i32(keys)
        n = keys.numel()
        out = self.ops.empty(n) if out is None else self._i32(out)
        pending = None

        def drain(p):
            lo, hi, rk, wk, index, send_counts, recv_counts = p
            if wk is not None:
                wk.wait()
            answers = self.ops.find(rk)
            back, _ = self._all_to_all(answers, recv_counts, send_counts, False)  # reverse route
            self.ops.unpermute(back, index, out[lo:hi])

        for lo, hi in self._chunks(n):
            pk, _, index, send_counts = self.ops.partition(self.alpha, self.beta, self.world, keys[lo:hi], None, True)
            recv_counts = self._exchange_counts(send_counts)
            rk, wk = self._all_to_all(pk, send_counts, recv_counts, True)
            if pending is not None:
                drain(pending)
            pending = (lo, hi, rk, wk, index, send_counts, recv_counts)
        if pending is not None:
            drain(pending)
        return out

    def inserted(self) -> int:
        t = self.ops.counts_tensor([self.ops.table.inserted()])
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def realized_load(self) -> float:
        return self.inserted() / (self.cfg.capacity * self.world)


class LocalShardedTable:
    """The single-process sharded handle of the C ABI (``bht_sharded_*``, csrc/sharded.cu): ``len(device_ids)`` shards,
    one ordinary table per entry (ids may repeat), routed by the same constants as :class:`ShardedTable`.  ``insert`` /
    ``find`` take one device tensor per shard — the slice that GPU contributes — and move the routed runs with peer
    copies; all owners work at the same time."""

    def __init__(self, cfg_per_shard, device_ids: Sequence[int]):
        self._lib = _lib.load()
        self.cfg = cfg_per_shard
        self.device_ids = [int(d) for d in device_ids]
        self._h = C.c_void_p()
        ids = (C.c_int32 * len(self.device_ids))(*self.device_ids)
        _check(self._lib.bht_sharded_create(C.byref(cfg_per_shard), len(self.device_ids), ids, C.byref(self._h)))
        a, b = C.c_uint64(), C.c_uint64()
        self._lib.bht_shard_constants(cfg_per_shard.seed, C.byref(a), C.byref(b))
        self.alpha, self.beta = a.value, b.value

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h:
            self._lib.bht_sharded_destroy(self._h)
            self._h = C.c_void_p()

    __del__ = close

    def __len__(self) -> int:
        return self._lib.bht_sharded_count(self._h)

    def shard(self, g: int) -> HashTable:
        """The table of shard g, borrowed (owned by this handle)."""
        h = C.c_void_p()
        _check(self._lib.bht_sharded_table(self._h, g, C.byref(h)))
        return HashTable._borrow(h, self.cfg, self.device_ids[g])

    def clear(self) -> None:
        _check(self._lib.bht_sharded_clear(self._h))

    def _slices(self, tensors, what: str):
        if len(tensors) != len(self.device_ids):
            raise ValueError(f"{what}: one tensor per shard expected")
        ptrs = (C.c_void_p * len(tensors))()
        ns = (C.c_uint64 * len(tensors))()
        for g, t in enumerate(tensors):
            if t is None:
                ptrs[g], ns[g] = None, 0
                continue
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.device.index == self.device_ids[g]):
                raise ValueError(f"{what}[{g}]: a tensor on cuda:{self.device_ids[g]} expected")
            if t.dtype not in (torch.int32, torch.uint32) or t.dim() != 1 or not t.is_contiguous():
                raise ValueError(f"{what}[{g}]: 1-D contiguous int32 / uint32 tensor expected")
            ptrs[g], ns[g] = t.data_ptr(), t.numel()
        return ptrs, ns

    def insert(self, keys: Sequence[torch.Tensor], values: Optional[Sequence[Optional[torch.Tensor]]] = None) -> BuildOutcome:
        for t in keys:
            if t is not None:
                torch.cuda.current_stream(t.device).synchronize()  # the handle works on its own streams
        kp, ns = self._slices(keys, "keys")
        vp = None
        if values is not None:
            vp, vns = self._slices(values, "values")
            for g in range(len(ns)):
                if values[g] is not None and vns[g] != ns[g]:
                    raise ValueError("insert: keys and values of a shard must have the same length")
        res = _lib.InsertResult()
        _check(self._lib.bht_sharded_insert(self._h, kp, vp, ns, C.byref(res)))
        return BuildOutcome(bool(res.success), res.inserted, res.failed, res.attempted, res.probes,
                            None if res.first_failed_key == _lib.EMPTY_KEY else res.first_failed_key)

    def find(self, keys: Sequence[torch.Tensor], want_stats: bool = False):
        for t in keys:
            if t is not None:
                torch.cuda.current_stream(t.device).synchronize()
        kp, ns = self._slices(keys, "keys")
        outs = [None if t is None else torch.empty_like(t) for t in keys]
        op, _ = self._slices(outs, "out")
        res = _lib.FindResult()
        _check(self._lib.bht_sharded_find(self._h, kp, op, ns, C.byref(res) if want_stats else None))
        if want_stats:
            from .table import FindStats
            return outs, FindStats(res.queries, res.hits, res.probes, res.value_sum)
        return outs
