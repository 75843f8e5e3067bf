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


class RoutingOverflow(RuntimeError):
    """A destination shard received more keys of one chunk than the fixed exchange segment holds (8 sigma above the
    mean of a uniform routing hash): the input is skewed against the routing hash.  Re-run with ``exact=True``."""


class CudaShardOps:
    """Per-rank device work of the sharded table, all through the C ABI."""

    supports_counted = True  # device-side chunk lengths (bht_build_feed_counted): the sync-free exchange

    def __init__(self, cfg, device: int):
        self.device = int(device)
        self.table = HashTable(cfg, self.device)
        self._lib = _lib.load()
        self.overflow = torch.zeros(1, dtype=torch.int32, device=self.torch_device)
        self.cuckoo = cfg.kind in (_lib_kind("bcht"), _lib_kind("1cht"))

    @property
    def torch_device(self):
        return torch.device("cuda", self.device)

    def empty(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=torch.int32, device=self.torch_device)

    def filled(self, n: int) -> torch.Tensor:
        """n words of 0xFFFFFFFF: the sentinel key / the "no slot" index of a padded exchange segment."""
        return torch.full((n,), -1, dtype=torch.int32, device=self.torch_device)

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

    def partition_fixed(self, alpha: int, beta: int, n_shards: int, keys: torch.Tensor, values: Optional[torch.Tensor],
                        want_index: bool, cap: int):
        """Routes into fixed segments of ``cap`` slots per destination, nothing copied to the host: returns
        (keys[n_shards * cap] padded with the sentinel, values or None, index padded with 0xFFFFFFFF or None,
        counts[n_shards] int64 on the device).  ``self.overflow`` is raised on the device when a segment was too small."""
        n = keys.numel()
        out_keys = self.filled(n_shards * cap)
        out_vals = self.empty(n_shards * cap) if values is not None else None
        index = self.filled(n_shards * cap) if want_index else None
        counts = torch.empty(n_shards, dtype=torch.int64, device=self.torch_device)
        _check(self._lib.bht_shard_partition_fixed(
            alpha, beta, n_shards, keys.data_ptr(), values.data_ptr() if values is not None else None, n, cap,
            out_keys.data_ptr(), out_vals.data_ptr() if out_vals is not None else None,
            index.data_ptr() if index is not None else None, counts.data_ptr(), self.overflow.data_ptr(), self.device,
            _stream_ptr(None, self.device)))
        return out_keys, out_vals, index, counts

    def unpermute(self, answers: torch.Tensor, index: torch.Tensor, out: torch.Tensor) -> None:
        _check(self._lib.bht_shard_unpermute(answers.data_ptr(), index.data_ptr(), answers.numel(), out.data_ptr(),
                                             self.device, _stream_ptr(None, self.device)))

    def insert(self, keys: torch.Tensor, values: torch.Tensor) -> BuildOutcome:
        return self.table.insert(keys, values)

    def build_begin(self, n_max: int) -> None:
        self.table.build_begin(n_max)

    def feed_counted(self, keys: torch.Tensor, values: torch.Tensor, cap: int, count: torch.Tensor) -> None:
        """One received segment: min(cap, count) pairs, ``count`` a one-element int64 device tensor."""
        _check(self._lib.bht_build_feed_counted(self.table._h, keys.data_ptr(), values.data_ptr(), cap, count.data_ptr(),
                                                _stream_ptr(None, self.device)))

    def build_feed(self, keys: torch.Tensor, values: torch.Tensor) -> None:
        self.table.build_feed(keys, values)

    def build_end(self) -> BuildOutcome:
        return self.table.build_end()

    def find_into(self, keys: torch.Tensor, out: torch.Tensor) -> None:
        self.table.find(keys, out)

    def find(self, keys: torch.Tensor) -> torch.Tensor:
        out = self.empty(keys.numel())
        self.table.find(keys, out)
        return out

    def counts_tensor(self, counts: Sequence[int]) -> torch.Tensor:
        return torch.tensor(list(counts), dtype=torch.int64, device=self.torch_device)


def _lib_kind(name: str) -> int:
    from .table import KINDS
    return KINDS[name]


class ShardedTable:
    """One logical table over ``world_size`` shards; call every method collectively on all ranks.

    Two exchanges.  The default one (cuckoo kinds) never synchronises with the host inside a call: every chunk is
    routed into fixed segments of ``cap`` slots per destination (the mean of a uniform routing hash + 8 sigma), sent
    with EQUAL-split all-to-alls, and the receive side learns the segment lengths on the device
    (bht_build_feed_counted) — one aggregate read at the end of the call (outcome + overflow flag).  The received
    chunks go through the table's chunked build, so a shard that qualifies takes the shared-memory-blocked build
    however many chunks it arrives in.  ``exact=True`` is the exchange with exact split sizes: one counts read per
    chunk, any skew."""

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
        self.phase_ms = {}  # bench.py: CUDA-event times of the phases of the last call (when record_phases is set)
        self.record_phases = False

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
        # every rank must issue the same number of collectives: agree on the max chunk count (the one host read
        # before the pipeline starts)
        mine = max(1, -(-n // self.chunk))
        t = self.ops.counts_tensor([mine, min(n, self.chunk)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        total, self._longest_chunk = (int(x) for x in t.tolist())
        return [(min(c * self.chunk, n), min((c + 1) * self.chunk, n)) for c in range(total)]

    def segment_cap(self, chunk_len: int) -> int:
        """Slots per destination of a fixed-segment exchange of ``chunk_len`` keys: mean + 8 sigma + 1024."""
        chunk_len = max(int(chunk_len), 4)
        if self.world == 1:
            return (chunk_len + 3) & ~3
        mean = chunk_len / self.world
        return min((chunk_len + 3) & ~3, (int(mean + 8.0 * mean ** 0.5) + 1024 + 3) & ~3)

    @staticmethod
    def _i32(x: torch.Tensor) -> torch.Tensor:
        return x.view(torch.int32) if x.dtype == torch.uint32 else x

    def _use_exact(self, exact: Optional[bool]) -> bool:
        if exact is None:
            return not (getattr(self.ops, "supports_counted", False) and getattr(self.ops, "cuckoo", False))
        return bool(exact)

    def _aggregate(self, totals, failed_key, overflow=None) -> BuildOutcome:
        t = self.ops.counts_tensor(list(totals))
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        flags = [-1 if failed_key is None else failed_key]
        fk = self.ops.counts_tensor(flags)
        if overflow is not None:
            fk = torch.cat([fk, overflow.to(torch.int64)])
        dist.all_reduce(fk, op=dist.ReduceOp.MAX, group=self.group)
        attempted, inserted, failed, probes = (int(x) for x in t.tolist())
        fl = [int(x) for x in fk.tolist()]
        if overflow is not None and fl[1] != 0:
            raise RoutingOverflow("sharded insert: a routing segment overflowed, its surplus pairs were not sent; "
                                  "clear the table and re-run with exact=True")
        return BuildOutcome(inserted == attempted, inserted, failed, attempted, probes, None if fl[0] < 0 else fl[0])

    # -- the hot path
    def insert(self, keys: torch.Tensor, values: torch.Tensor, exact: Optional[bool] = None) -> BuildOutcome:
        """Routes this rank's (key, value) pairs to their owners and bulk-inserts what this rank owns.
        Returns the outcome aggregated over all ranks."""
        keys, values = self._i32(keys), self._i32(values)
        if self.world == 1 and exact is None and hasattr(self.ops, "build_feed"):
            # one shard owns every key: nothing to route, the chunks go straight into the chunked build
            self.ops.build_begin(self.cfg.capacity)
            for lo, hi in self._chunks(keys.numel()):
                self.ops.build_feed(keys[lo:hi], values[lo:hi])
            o = self.ops.build_end()
            return self._aggregate([o.attempted, o.inserted, o.failed, o.probes], o.failed_key)
        if self._use_exact(exact):
            return self._insert_exact(keys, values)
        chunks = self._chunks(keys.numel())
        cap = self.segment_cap(self._longest_chunk)  # the same on every rank
        self.ops.overflow.zero_()
        self.ops.build_begin(self.cfg.capacity)
        pending = None

        def drain(p):
            rk, rv, rc, works = p
            for w in works:
                w.wait()
            for src in range(self.world):
                self.ops.feed_counted(rk[src * cap:(src + 1) * cap], rv[src * cap:(src + 1) * cap], cap, rc[src:src + 1])

        for lo, hi in chunks:
            sk, sv, _, counts = self.ops.partition_fixed(self.alpha, self.beta, self.world, keys[lo:hi], values[lo:hi], False, cap)
            rc = torch.empty_like(counts)
            rk, rv = self.ops.empty(self.world * cap), self.ops.empty(self.world * cap)
            works = [dist.all_to_all_single(rc, counts, group=self.group, async_op=True),
                     dist.all_to_all_single(rk, sk, group=self.group, async_op=True),
                     dist.all_to_all_single(rv, sv, group=self.group, async_op=True)]
            if pending is not None:
                drain(pending)  # the previous chunk's partition pass runs under this chunk's exchange
            pending = (rk, rv, rc, works)
        if pending is not None:
            drain(pending)
        o = self.ops.build_end()  # the one host read of the call
        return self._aggregate([o.attempted, o.inserted, o.failed, o.probes], o.failed_key, self.ops.overflow)

    def _insert_exact(self, keys: torch.Tensor, values: torch.Tensor) -> BuildOutcome:
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
        return self._aggregate(totals, failed_key)

    def find(self, keys: torch.Tensor, out: Optional[torch.Tensor] = None, exact: Optional[bool] = None) -> torch.Tensor:
        """Answers this rank's queries in the caller's order: out[i] = value or EMPTY_VALUE."""
        keys = self._i32(keys)
        n = keys.numel()
        out = self.ops.empty(n) if out is None else self._i32(out)
        if self.world == 1 and exact is None and hasattr(self.ops, "find_into"):
            for lo, hi in self._chunks(n):
                self.ops.find_into(keys[lo:hi], out[lo:hi])
            return out
        if self._use_exact(exact):
            return self._find_exact(keys, out)
        chunks = self._chunks(n)
        cap = self.segment_cap(self._longest_chunk)  # the same on every rank
        self.ops.overflow.zero_()
        # three stages in flight: the keys of chunk i + 1 travel while chunk i is probed and the answers of chunk i - 1 travel back
        arriving, returning = None, None

        def probe(p):
            lo, hi, rk, wk, index = p
            wk.wait()
            answers = self.ops.find(rk)  # padding slots hold the sentinel key: answered EMPTY without a probe
            back = self.ops.empty(self.world * cap)
            wb = dist.all_to_all_single(back, answers, group=self.group, async_op=True)  # reverse route, same equal splits
            return lo, hi, back, wb, index, answers

        def deliver(p):
            lo, hi, back, wb, index, _answers = p
            wb.wait()
            self.ops.unpermute(back, index, out[lo:hi])  # padding slots carry the index 0xFFFFFFFF: skipped

        for lo, hi in chunks:
            sk, _, index, _counts = self.ops.partition_fixed(self.alpha, self.beta, self.world, keys[lo:hi], None, True, cap)
            rk = self.ops.empty(self.world * cap)
            wk = dist.all_to_all_single(rk, sk, group=self.group, async_op=True)
            probed = probe(arriving) if arriving is not None else None
            if returning is not None:
                deliver(returning)
            arriving, returning = (lo, hi, rk, wk, index), probed
        probed = probe(arriving) if arriving is not None else None
        if returning is not None:
            deliver(returning)
        if probed is not None:
            deliver(probed)
        flag = self.ops.overflow.to(torch.int64)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
        if int(flag.item()) != 0:  # the one host read of the call
            raise RoutingOverflow("sharded find: a routing segment overflowed; re-run with exact=True")
        return out

    def _find_exact(self, keys: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        pending = None

        def drain(p):
            lo, hi, rk, wk, index, send_counts, recv_counts = p
            if wk is not None:
                wk.wait()
            answers = self.ops.find(rk)
            back, _ = self._all_to_all(answers, recv_counts, send_counts, False)  # reverse route
            self.ops.unpermute(back, index, out[lo:hi])

        for lo, hi in self._chunks(keys.numel()):
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
