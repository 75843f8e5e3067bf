"""Host-side mirror of the reference table API (proj/include/bht/table.hpp, core.hpp) over the C ABI.

Same names and argument meaning as the reference: ``make_config``, ``hash_table`` (``HashTable``),
``build``, ``insert`` / ``find`` (the bulk forms of ``insert_pair`` / ``find_key``), ``realized_load``,
``occupied_slots``, ``dump_store``, ``slot_at``, ``poke_slot``.  Error behaviour follows the reference's
exceptions (core.cpp:40-60, table.cpp:15-17,22-23,225):

    std::invalid_argument -> ValueError            std::logic_error   -> KindMismatchError
    capacity exceeded     -> CapacityError(ValueError)   std::runtime_error -> OSError (file I/O)

A failed insertion is not an error; it is reported in ``BuildOutcome`` as in ``build_outcome``
(table.hpp:115-120).

Key / value / answer arrays may be CUDA tensors on the table's device (zero-copy, stream-ordered) or
host arrays (numpy / CPU tensors; staged over PCIe by the library).  torch is used for device memory and
streams only; every table operation is a call into lib/libbht_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import Config, FindResult, InsertResult

KINDS = {"1cht": 0, "one_cht": 0, "bcht": 1, "bp2ht": 2, "iht": 3}
KIND_NAMES = {0: "1cht", 1: "bcht", 2: "bp2ht", 3: "iht"}
EMPTY_KEY = EMPTY_VALUE = _lib.EMPTY_KEY
EMPTY_SLOT = _lib.EMPTY_SLOT
OP_INSERT, OP_FIND = 0, 1


class KindMismatchError(RuntimeError):
    """std::logic_error of require_kind (table.cpp:15-17)."""


class CapacityError(ValueError):
    """std::invalid_argument "build: key set exceeds table capacity" (table.cpp:225)."""


class CudaError(RuntimeError):
    pass


def _check(status: int) -> None:
    if status == _lib.OK:
        return
    msg = _lib.last_error()
    if status == _lib.INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == _lib.KIND_MISMATCH:
        raise KindMismatchError(msg)
    if status == _lib.CAPACITY_EXCEEDED:
        raise CapacityError(msg)
    if status == _lib.IO_ERROR:
        raise OSError(msg)
    raise CudaError(msg)


def kind_id(kind) -> int:
    if isinstance(kind, str):
        if kind not in KINDS:
            raise ValueError(f"unknown table kind {kind!r}")  # parse_table_kind (core.cpp:20-26)
        return KINDS[kind]
    return int(kind)


# ---- configuration (core.hpp / core.cpp) ----------------------------------------------------------------------

def make_config(kind, n_keys: int, lf: float, bucket_size: int, threshold: Optional[int] = None, seed: int = 0,
                max_chain: Optional[int] = None) -> Config:
    """make_config (core.hpp:85-91, core.cpp:33-68), bit-exact: m = ceil(n/(lf*b)), same hash-constant draw."""
    cfg = Config()
    _check(_lib.load().bht_make_config(kind_id(kind), n_keys, float(lf), bucket_size,
                                       -1 if threshold is None else threshold, seed,
                                       -1 if max_chain is None else max_chain, C.byref(cfg)))
    return cfg


def craft_config(kind, num_buckets: int, bucket_size: int, hashes, threshold: int = 0, max_chain: int = 8,
                 seed: int = 1) -> Config:
    """A handcrafted configuration (the reference tests' ``craft``, proj/tests/test_table.cpp:15-28)."""
    cfg = Config()
    cfg.kind = kind_id(kind)
    cfg.num_buckets = num_buckets
    cfg.bucket_size = bucket_size
    cfg.capacity = num_buckets * bucket_size
    cfg.n_hashes = len(hashes)
    for i, (a, b, r) in enumerate(hashes[:_lib.MAX_HASHES]):
        cfg.alpha[i], cfg.beta[i], cfg.range[i] = a, b, r
    cfg.threshold = threshold
    cfg.max_chain = max_chain
    cfg.seed = seed
    return cfg


def hash_count(kind) -> int:
    return _lib.load().bht_hash_count(kind_id(kind))


def default_max_chain(n_keys: int) -> int:
    return _lib.load().bht_default_max_chain(n_keys)


def mix_seed(seed: int, stream: int) -> int:
    return _lib.load().bht_mix_seed(seed, stream)


def bucket_index(alpha: int, beta: int, rng: int, key: int) -> int:
    """bucket_index (hash.hpp:21-23) through the division-free host twin of the device hash stage."""
    r = _lib.load().bht_bucket_index_host(alpha, beta, rng, key)
    if r == 0xFFFFFFFFFFFFFFFF:
        raise ValueError(_lib.last_error())
    return r


def value_for_key(key: int) -> int:
    return _lib.load().bht_value_for_key(key)


def predict_sectors(kind, bucket_size: int, mean_probes: float, op: int) -> float:
    """predict_sectors (sector_model.hpp:26-31); op = OP_INSERT | OP_FIND."""
    return _lib.load().bht_predict_sectors(kind_id(kind), bucket_size, float(mean_probes), op)


def pack_pair(key: int, value: int) -> int:
    return ((value & 0xFFFFFFFF) << 32) | (key & 0xFFFFFFFF)  # core.hpp:35-37


def unpack_slot(slot: int) -> Tuple[int, int]:
    return slot & 0xFFFFFFFF, (slot >> 32) & 0xFFFFFFFF  # core.hpp:39-41


# ---- array plumbing ---------------------------------------------------------------------------------------------

def _as_u32(x, name: str):
    """Returns (pointer, n, mem_space, keepalive) for a 1-D array of 32-bit words."""
    if isinstance(x, torch.Tensor):
        if x.dtype not in (torch.uint32, torch.int32):
            raise ValueError(f"{name}: tensor dtype must be uint32 or int32, got {x.dtype}")
        if x.dim() != 1 or not x.is_contiguous():
            raise ValueError(f"{name}: tensor must be 1-D and contiguous")
        space = _lib.MEM_DEVICE if x.is_cuda else _lib.MEM_HOST
        return x.data_ptr(), x.numel(), space, x
    a = np.ascontiguousarray(x)
    if a.dtype not in (np.uint32, np.int32):
        raise ValueError(f"{name}: array dtype must be uint32 or int32, got {a.dtype}")
    if a.ndim != 1:
        raise ValueError(f"{name}: array must be 1-D")
    return a.ctypes.data, a.size, _lib.MEM_HOST, a


def _stream_ptr(stream, device: int) -> int:
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def values_for_keys(keys):
    """value_for_key (keygen.hpp:23-26) over an array, in the array's own memory space."""
    if isinstance(keys, torch.Tensor):
        k = keys.view(torch.int32)
        v = torch.bitwise_xor(k, 0x5A5A5A5A)
        v = torch.where(v == -1, torch.full_like(v, 0x7FFFFFFF), v)
        return v.view(torch.uint32)
    k = np.asarray(keys, dtype=np.uint32)
    v = k ^ np.uint32(0x5A5A5A5A)
    v[v == 0xFFFFFFFF] = 0x7FFFFFFF
    return v


@dataclass
class BuildOutcome:
    """build_outcome (table.hpp:115-120) for one bulk insert."""
    success: bool
    inserted: int
    failed: int
    attempted: int
    probes: int
    failed_key: Optional[int]

    @property
    def mean_probes(self) -> float:
        return self.probes / self.attempted if self.attempted else 0.0


@dataclass
class FindStats:
    queries: int
    hits: int
    probes: int
    value_sum: int

    @property
    def mean_probes(self) -> float:
        return self.probes / self.queries if self.queries else 0.0


class _DeviceStoreView:
    """__cuda_array_interface__ over the table's slot store (int64 words; torch lacks uint64 indexing)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 2}


class HashTable:
    """``class hash_table`` (table.hpp:28-80) with its slot store in device memory."""

    def __init__(self, cfg: Config, device: Optional[int] = None):
        self._lib = _lib.load()
        self._h = C.c_void_p()
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = int(device)
        self._cfg = cfg.copy()
        _check(self._lib.bht_create(C.byref(self._cfg), self.device, C.byref(self._h)))

    @classmethod
    def _adopt(cls, handle, cfg: Config, device: int) -> "HashTable":
        """Wraps a table created by the library (bht_build)."""
        self = cls.__new__(cls)
        self._lib = _lib.load()
        self._h = handle
        self.device = device
        self._cfg = cfg.copy()
        return self

    @classmethod
    def _borrow(cls, handle, cfg: Config, device: int) -> "HashTable":
        """Wraps a table owned by someone else (a shard of bht_sharded): close() does not destroy it."""
        self = cls._adopt(handle, cfg, device)
        self._borrowed = True
        return self

    # -- lifetime
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h:
            if not getattr(self, "_borrowed", False):
                self._lib.bht_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- accessors (table.hpp:32-47)
    def config(self) -> Config:
        return self._cfg

    @property
    def kind(self) -> str:
        return KIND_NAMES[self._cfg.kind]

    def num_buckets(self) -> int:
        return self._cfg.num_buckets

    def bucket_size(self) -> int:
        return self._cfg.bucket_size

    def capacity(self) -> int:
        return self._cfg.capacity

    def bucket_of(self, i: int, key: int) -> int:
        a, b, r = self._cfg.hashes[i]
        return bucket_index(a, b, r, key)

    def inserted(self) -> int:
        ins, cap = C.c_uint64(), C.c_uint64()
        _check(self._lib.bht_load_factor(self._h, C.byref(ins), C.byref(cap)))
        return ins.value

    def realized_load(self) -> float:
        return self.inserted() / self._cfg.capacity

    def occupied_slots(self, stream=None) -> int:
        out = C.c_uint64()
        _check(self._lib.bht_count_occupied(self._h, C.byref(out), _stream_ptr(stream, self.device)))
        return out.value

    def count_inadmissible(self, stream=None) -> int:
        """check_admissibility (oracle.cpp:40-54) evaluated on the device."""
        out = C.c_uint64()
        _check(self._lib.bht_count_inadmissible(self._h, C.byref(out), _stream_ptr(stream, self.device)))
        return out.value

    def clear(self, stream=None) -> None:
        _check(self._lib.bht_clear(self._h, _stream_ptr(stream, self.device)))

    def set_iht_prose_fallback(self, enabled: bool) -> None:
        _check(self._lib.bht_set_iht_prose_fallback(self._h, int(bool(enabled))))

    def set_blocked_insert(self, mode) -> None:
        """Blocked builds of device-resident inserts: 0 / False = never (caller order), 1 / True = when the sizes
        make it pay (default: shared-memory-blocked for bcht, L2-routed for 1cht), 2 = always the L2-routed build,
        3 = always the shared-memory-blocked build.  bp2ht / iht always insert in caller order; for them modes 1 (stores
        of 192 MB and more) and 3 take the loads from the per-bucket counter array (csrc/insert_claim.cu), mode 0 reads
        the candidate buckets."""
        _check(self._lib.bht_set_blocked_insert(self._h, int(mode)))

    def last_build_schedule(self) -> int:
        """0 = caller order, 2 = L2-routed, 3 = shared-memory-blocked: how the last insert / chunked build ran."""
        return int(self._lib.bht_last_build_schedule(self._h))

    # -- the hot path
    def insert(self, keys, values=None, n: Optional[int] = None, stream=None, want_result: bool = True,
               as_kind=None) -> Optional[BuildOutcome]:
        """Bulk insert_pair (table.hpp:103-104) / build()'s loop (table.cpp:224-271).

        ``values=None`` derives value_for_key(k) as ``build`` does (table.cpp:234).  ``as_kind`` selects the
        reference's per-variant entry point (bcht_insert / bp2ht_insert / iht_insert) and its kind check.
        """
        kp, kn, kspace, _k = _as_u32(keys, "keys")
        if values is None:  # NULL values: the library pairs every key with value_for_key(key) on the device
            vp, vn, vspace, _v = None, kn, kspace, None
        else:
            vp, vn, vspace, _v = _as_u32(values, "values")
        if kspace != vspace:
            raise ValueError("insert: keys and values must live in the same memory space")
        n = kn if n is None else int(n)
        if n > kn or n > vn:
            raise ValueError("insert: n exceeds the array length")
        res = InsertResult()
        rp = C.byref(res) if want_result else None
        sp = _stream_ptr(stream, self.device)
        if as_kind is None:
            _check(self._lib.bht_insert(self._h, kp, vp, n, kspace, rp, sp))
        else:
            _check(self._lib.bht_insert_as(self._h, kind_id(as_kind), kp, vp, n, kspace, rp, sp))
        if not want_result:
            return None
        return BuildOutcome(bool(res.success), res.inserted, res.failed, res.attempted, res.probes,
                            None if res.first_failed_key == EMPTY_KEY else res.first_failed_key)

    # -- a build whose pairs arrive in chunks (bht_build_begin / _feed / _end)
    def build_begin(self, n_max: int, stream=None) -> None:
        """Opens a chunked build of at most ``n_max`` pairs (the receive side of a sharded build)."""
        _check(self._lib.bht_build_begin(self._h, int(n_max), _stream_ptr(stream, self.device)))

    def build_feed(self, keys, values=None, n: Optional[int] = None, stream=None) -> None:
        """Adds a device-resident chunk; ``values=None`` pairs every key with value_for_key(key)."""
        kp, kn, kspace, _k = _as_u32(keys, "keys")
        if kspace != _lib.MEM_DEVICE:
            raise ValueError("build_feed: chunks must be device-resident")
        vp = None
        n = kn if n is None else int(n)
        if values is not None:
            vp, vn, vspace, _v = _as_u32(values, "values")
            if vspace != _lib.MEM_DEVICE or vn < n:
                raise ValueError("build_feed: values must be device-resident and at least n long")
        if n > kn:
            raise ValueError("build_feed: n exceeds the array length")
        _check(self._lib.bht_build_feed(self._h, kp, vp, n, _stream_ptr(stream, self.device)))

    def build_end(self, stream=None, want_result: bool = True) -> Optional[BuildOutcome]:
        res = InsertResult()
        _check(self._lib.bht_build_end(self._h, C.byref(res) if want_result else None, _stream_ptr(stream, self.device)))
        if not want_result:
            return None
        return BuildOutcome(bool(res.success), res.inserted, res.failed, res.attempted, res.probes,
                            None if res.first_failed_key == EMPTY_KEY else res.first_failed_key)

    def last_insert_result(self, stream=None) -> BuildOutcome:
        res = InsertResult()
        _check(self._lib.bht_last_insert_result(self._h, C.byref(res), _stream_ptr(stream, self.device)))
        return BuildOutcome(bool(res.success), res.inserted, res.failed, res.attempted, res.probes,
                            None if res.first_failed_key == EMPTY_KEY else res.first_failed_key)

    def set_repair(self, enabled: bool) -> None:
        """cuckoo kinds: the few pairs a launch dropped at the chain cap are inserted once more, one at a time, as the
        reference inserts every pair (on by default; off = the raw outcome of the concurrent walks)."""
        _check(self._lib.bht_set_repair(self._h, int(bool(enabled))))

    def set_tail_throttle(self, enabled: bool) -> None:
        """cuckoo kinds: insert the pairs that arrive beyond load 0.98 with few keys in flight — build success at load
        factor 0.99 closer to the reference's (~80 % instead of ~50 %; reference 90 %) for 2.5x the build time.  Off by
        default: retrying a failed build is cheaper."""
        _check(self._lib.bht_set_tail_throttle(self._h, int(bool(enabled))))

    def last_insert_phases(self):
        """(prepare_ms, probe_ms) of the last device-resident insert: routing / binning passes, then the bulk-insert
        kernel, timed with CUDA events inside the library."""
        a, b = C.c_float(), C.c_float()
        _check(self._lib.bht_last_insert_phases(self._h, C.byref(a), C.byref(b)))
        return float(a.value), float(b.value)

    def failed_keys(self, max_keys: int = 1 << 20) -> np.ndarray:
        buf = np.empty(max_keys, dtype=np.uint32)
        cnt = C.c_uint64()
        _check(self._lib.bht_failed_keys(self._h, buf.ctypes.data, max_keys, C.byref(cnt)))
        return buf[:min(cnt.value, max_keys)].copy()

    def _find(self, fn, keys, out, n, stream, want_stats, as_kind=None):
        kp, kn, kspace, _k = _as_u32(keys, "keys")
        n = kn if n is None else int(n)
        if n > kn:
            raise ValueError("find: n exceeds the array length")
        if out is None:
            if isinstance(keys, torch.Tensor):
                out = torch.empty(n, dtype=torch.uint32, device=keys.device, pin_memory=not keys.is_cuda and torch.cuda.is_available())
            else:
                out = np.empty(n, dtype=np.uint32)
        op, on, ospace, _o = _as_u32(out, "out")
        if ospace != kspace:
            raise ValueError("find: keys and out must live in the same memory space")
        if on < n:
            raise ValueError("find: out is shorter than n")
        res = FindResult()
        rp = C.byref(res) if want_stats else None
        sp = _stream_ptr(stream, self.device)
        if as_kind is None:
            _check(fn(self._h, kp, op, n, kspace, rp, sp))
        else:
            _check(fn(self._h, kind_id(as_kind), kp, op, n, kspace, rp, sp))
        if want_stats:
            return out, FindStats(res.queries, res.hits, res.probes, res.value_sum)
        return out

    def find(self, keys, out=None, n: Optional[int] = None, stream=None, want_stats: bool = False, as_kind=None):
        """Bulk find_key (table.hpp:105): out[i] = value or EMPTY_VALUE (0xFFFFFFFF) when absent."""
        if as_kind is not None:
            return self._find(self._lib.bht_find_as, keys, out, n, stream, want_stats, as_kind)
        return self._find(self._lib.bht_find, keys, out, n, stream, want_stats)

    def find_exhaustive(self, keys, out=None, n: Optional[int] = None, stream=None, want_stats: bool = False):
        """bcht_find_no_early_exit (oracle.cpp:56-63): probes every candidate bucket."""
        return self._find(self._lib.bht_find_exhaustive, keys, out, n, stream, want_stats)

    # -- store access (table.hpp:53-56, table.cpp:41-51)
    def download_store(self, stream=None) -> np.ndarray:
        out = np.empty(self._cfg.capacity, dtype=np.uint64)
        _check(self._lib.bht_download_store(self._h, out.ctypes.data, _stream_ptr(stream, self.device)))
        return out

    def upload_store(self, store, stream=None) -> None:
        a = np.ascontiguousarray(store, dtype=np.uint64)
        if a.size != self._cfg.capacity:
            raise ValueError("upload_store: store length must equal capacity")
        _check(self._lib.bht_upload_store(self._h, a.ctypes.data, _stream_ptr(stream, self.device)))

    def dump_store(self, path: str) -> None:
        _check(self._lib.bht_dump_store(self._h, str(path).encode()))

    def device_store(self) -> torch.Tensor:
        """Zero-copy int64 view of the slot store (bucket-major, b consecutive slots per bucket)."""
        ptr = self._lib.bht_device_store(self._h)
        with torch.cuda.device(self.device):
            return torch.as_tensor(_DeviceStoreView(ptr, self._cfg.capacity), device=f"cuda:{self.device}")

    def slot_at(self, index: int) -> int:
        if not 0 <= index < self._cfg.capacity:
            raise IndexError(index)
        return int(self.device_store()[index].item()) & EMPTY_SLOT

    def poke_slot(self, index: int, slot: int) -> None:
        """Raw slot write for fault injection (table.hpp:54-56); does not touch the inserted counter."""
        if not 0 <= index < self._cfg.capacity:
            raise IndexError(index)
        signed = slot - (1 << 64) if slot >= (1 << 63) else slot
        self.device_store()[index] = signed
        torch.cuda.synchronize(self.device)


hash_table = HashTable  # the reference's class name


def build(keys, cfg: Config, values=None, device: Optional[int] = None, iht_prose_fallback: bool = False,
          stream=None) -> Tuple[HashTable, BuildOutcome]:
    """build(keys, cfg, opts) (table.hpp:125-127, table.cpp:224-276) as ONE bulk device insert.

    Unlike the reference, which stops at the first failed key, every key is attempted; ``success`` still means
    inserted == len(keys).  Raises CapacityError when len(keys) > capacity, before touching the device store.
    """
    kp, kn, kspace, _k = _as_u32(keys, "keys")
    if values is None:  # the reference's signature: the library pairs key k with value_for_key(k) on the device
        vp, vn, vspace, _v = None, kn, kspace, None
    else:
        vp, vn, vspace, _v = _as_u32(values, "values")
    if kspace != vspace or kn != vn:
        raise ValueError("build: keys and values must have the same length and memory space")
    if device is None:
        device = keys.device.index if isinstance(keys, torch.Tensor) and keys.is_cuda else (
            torch.cuda.current_device() if torch.cuda.is_available() else 0)
    handle = C.c_void_p()
    res = InsertResult()
    _check(_lib.load().bht_build(C.byref(cfg), int(device), kp, vp, kn, kspace, int(bool(iht_prose_fallback)),
                                 C.byref(handle), C.byref(res), _stream_ptr(stream, int(device))))
    table = HashTable._adopt(handle, cfg, int(device))
    outcome = BuildOutcome(bool(res.success), res.inserted, res.failed, res.attempted, res.probes,
                           None if res.first_failed_key == EMPTY_KEY else res.first_failed_key)
    return table, outcome


def hash_keys(alpha: int, beta: int, rng: int, keys, device: Optional[int] = None, stream=None):
    """The device hash stage in isolation: out[i] = bucket_index({alpha, beta, rng}, keys[i])."""
    lib = _lib.load()
    kp, n, space, _k = _as_u32(keys, "keys")
    if isinstance(keys, torch.Tensor) and keys.is_cuda:
        device = keys.device.index
        out = torch.empty(n, dtype=torch.uint32, device=keys.device)
    else:
        device = 0 if device is None else device
        out = np.empty(n, dtype=np.uint32)
    op = out.data_ptr() if isinstance(out, torch.Tensor) else out.ctypes.data
    _check(lib.bht_hash_keys(alpha, beta, rng, kp, op, n, space, device, _stream_ptr(stream, device)))
    return out


def generate_unique_keys(seed: int, offset: int, n: int, device: Optional[int] = None, with_values: bool = True,
                         stream=None):
    """Device-side synthetic workload: keys = a bijection of the counters [offset, offset+n) over [0, 2^32-2]."""
    lib = _lib.load()
    device = torch.cuda.current_device() if device is None else device
    keys = torch.empty(n, dtype=torch.uint32, device=f"cuda:{device}")
    vals = torch.empty(n, dtype=torch.uint32, device=f"cuda:{device}") if with_values else None
    _check(lib.bht_generate_unique_keys(seed, offset, n, keys.data_ptr(), vals.data_ptr() if with_values else None,
                                        device, _stream_ptr(stream, device)))
    return (keys, vals) if with_values else keys


def reload_tuning() -> None:
    """Re-reads the BHT_* tuning environment variables (the library reads them once per process)."""
    _lib.load().bht_reload_tuning()


def kernel_launch_count() -> int:
    return _lib.load().bht_kernel_launch_count()
