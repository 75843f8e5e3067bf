"""ctypes binding of the C ABI in include/bht_b200.h (lib/libbht_b200.so).

This is the only way the Python host layer reaches the device: there is no CPU or PyTorch fallback.
If the shared library has not been built the import fails loudly (``BhtLibraryMissing``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# BHT_B200_LIB: another build of the same library (A/B runs of tuning macros, csrc/Makefile VARIANT=...)
LIB_PATH = os.environ.get("BHT_B200_LIB") or os.path.join(HERE, "lib", "libbht_b200.so")

OK, INVALID_ARGUMENT, KIND_MISMATCH, CAPACITY_EXCEEDED, CUDA_ERROR, COMM_ERROR, IO_ERROR = range(7)
MEM_DEVICE, MEM_HOST = 0, 1
EMPTY_KEY = EMPTY_VALUE = 0xFFFFFFFF
EMPTY_SLOT = 0xFFFFFFFFFFFFFFFF
HASH_PRIME = 4294967291
MAX_HASHES = 4


class BhtLibraryMissing(ImportError):
    pass


class Config(C.Structure):
    """bht_config: the plain-data image of the reference ``table_config`` (core.hpp:66-77)."""

    _fields_ = [
        ("kind", C.c_int32),
        ("bucket_size", C.c_uint32),
        ("num_buckets", C.c_uint64),
        ("capacity", C.c_uint64),
        ("n_hashes", C.c_uint32),
        ("threshold", C.c_uint32),
        ("max_chain", C.c_uint32),
        ("reserved", C.c_uint32),
        ("seed", C.c_uint64),
        ("alpha", C.c_uint64 * MAX_HASHES),
        ("beta", C.c_uint64 * MAX_HASHES),
        ("range", C.c_uint64 * MAX_HASHES),
    ]

    def copy(self) -> "Config":
        c = Config()
        C.memmove(C.byref(c), C.byref(self), C.sizeof(Config))
        return c

    @property
    def hashes(self):
        return [(int(self.alpha[i]), int(self.beta[i]), int(self.range[i])) for i in range(self.n_hashes)]

    def __repr__(self):
        return (f"Config(kind={self.kind}, m={self.num_buckets}, b={self.bucket_size}, capacity={self.capacity}, "
                f"threshold={self.threshold}, max_chain={self.max_chain}, seed={self.seed}, hashes={self.hashes})")


class InsertResult(C.Structure):
    """bht_insert_result: the image of ``build_outcome`` (table.hpp:115-120)."""

    _fields_ = [
        ("attempted", C.c_uint64),
        ("inserted", C.c_uint64),
        ("failed", C.c_uint64),
        ("probes", C.c_uint64),
        ("first_failed_key", C.c_uint32),
        ("success", C.c_uint32),
    ]


class FindResult(C.Structure):
    _fields_ = [
        ("queries", C.c_uint64),
        ("hits", C.c_uint64),
        ("probes", C.c_uint64),
        ("value_sum", C.c_uint64),
    ]


_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol include/bht_b200.h declares
SIGNATURES = {
    "bht_make_config": (C.c_int, [C.c_int32, C.c_uint64, C.c_double, C.c_uint32, C.c_int64, C.c_uint64, C.c_int64, C.POINTER(Config)]),
    "bht_hash_count": (C.c_uint32, [C.c_int32]),
    "bht_default_max_chain": (C.c_uint32, [C.c_uint64]),
    "bht_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "bht_bucket_index_host": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32]),
    "bht_value_for_key": (C.c_uint32, [C.c_uint32]),
    "bht_predict_sectors": (C.c_double, [C.c_int32, C.c_uint32, C.c_double, C.c_int32]),
    "bht_create": (C.c_int, [C.POINTER(Config), C.c_int32, C.POINTER(_vp)]),
    "bht_destroy": (C.c_int, [_vp]),
    "bht_clear": (C.c_int, [_vp, _vp]),
    "bht_get_config": (C.c_int, [_vp, C.POINTER(Config)]),
    "bht_device_of": (C.c_int32, [_vp]),
    "bht_insert": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int32, C.POINTER(InsertResult), _vp]),
    "bht_build": (C.c_int, [C.POINTER(Config), C.c_int32, _vp, _vp, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(_vp),
                            C.POINTER(InsertResult), _vp]),
    "bht_insert_as": (C.c_int, [_vp, C.c_int32, _vp, _vp, C.c_uint64, C.c_int32, C.POINTER(InsertResult), _vp]),
    "bht_build_begin": (C.c_int, [_vp, C.c_uint64, _vp]),
    "bht_build_feed": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _vp]),
    "bht_build_end": (C.c_int, [_vp, C.POINTER(InsertResult), _vp]),
    "bht_build_feed_counted": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _vp, _vp]),
    "bht_shard_partition_fixed": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, _vp, _vp, C.c_uint64, C.c_uint64, _vp, _vp, _vp, _vp, _vp,
                                            C.c_int32, _vp]),
    "bht_find": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int32, C.POINTER(FindResult), _vp]),
    "bht_find_as": (C.c_int, [_vp, C.c_int32, _vp, _vp, C.c_uint64, C.c_int32, C.POINTER(FindResult), _vp]),
    "bht_find_exhaustive": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int32, C.POINTER(FindResult), _vp]),
    "bht_last_insert_result": (C.c_int, [_vp, C.POINTER(InsertResult), _vp]),
    "bht_failed_keys": (C.c_int, [_vp, _vp, C.c_uint64, _u64p]),
    "bht_set_iht_prose_fallback": (C.c_int, [_vp, C.c_int32]),
    "bht_set_blocked_insert": (C.c_int, [_vp, C.c_int32]),
    "bht_last_build_schedule": (C.c_int32, [_vp]),
    "bht_set_tail_throttle": (C.c_int, [_vp, C.c_int32]),
    "bht_set_repair": (C.c_int, [_vp, C.c_int32]),
    "bht_last_insert_phases": (C.c_int, [_vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "bht_load_factor": (C.c_int, [_vp, _u64p, _u64p]),
    "bht_count_occupied": (C.c_int, [_vp, _u64p, _vp]),
    "bht_download_store": (C.c_int, [_vp, _vp, _vp]),
    "bht_upload_store": (C.c_int, [_vp, _vp, _vp]),
    "bht_dump_store": (C.c_int, [_vp, C.c_char_p]),
    "bht_count_inadmissible": (C.c_int, [_vp, _u64p, _vp]),
    "bht_device_store": (C.c_void_p, [_vp]),
    "bht_hash_keys": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp, C.c_uint64, C.c_int32, C.c_int32, _vp]),
    "bht_shard_of_host": (C.c_uint32, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]),
    "bht_shard_partition": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, _vp, _vp, C.c_uint64, _vp, _vp, _vp, _u64p, C.c_int32, _vp]),
    "bht_shard_unpermute": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_int32, _vp]),
    "bht_shard_constants": (None, [C.c_uint64, _u64p, _u64p]),
    "bht_sharded_create": (C.c_int, [C.POINTER(Config), C.c_uint32, C.POINTER(C.c_int32), C.POINTER(_vp)]),
    "bht_sharded_destroy": (C.c_int, [_vp]),
    "bht_sharded_count": (C.c_uint32, [_vp]),
    "bht_sharded_table": (C.c_int, [_vp, C.c_uint32, C.POINTER(_vp)]),
    "bht_sharded_clear": (C.c_int, [_vp]),
    "bht_sharded_insert": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), _u64p, C.POINTER(InsertResult)]),
    "bht_sharded_find": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), _u64p, C.POINTER(FindResult)]),
    "bht_generate_unique_keys": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp, C.c_int32, _vp]),
    "bht_unique_key_host": (C.c_uint32, [C.c_uint64, C.c_uint32]),
    "bht_synthetic_value_host": (C.c_uint32, [C.c_uint64, C.c_uint32]),
    "bht_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "bht_host_free": (C.c_int, [_vp]),
    "bht_last_error_string": (C.c_char_p, []),
    "bht_generate_keys": (C.c_int, [C.c_uint64, C.c_uint64, _vp, C.c_int32, C.c_int32, _vp]),
    "bht_generate_queries": (C.c_int, [_vp, C.c_uint64, C.c_int32, C.c_double, C.c_uint64, C.c_uint64, _vp, _vp, _vp, C.c_int32]),
    "bht_save_keys": (C.c_int, [C.c_char_p, _vp, C.c_uint64]),
    "bht_load_keys": (C.c_int, [C.c_char_p, _vp, C.c_uint64, _u64p]),
    "bht_version_string": (C.c_char_p, []),
    "bht_reload_tuning": (None, []),
    "bht_kernel_launch_count": (C.c_uint64, []),
    "bht_sizeof_config": (C.c_size_t, []),
}

_lib = None


def load() -> C.CDLL:
    """Loads lib/libbht_b200.so once and types every entry point. Raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BhtLibraryMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_2108_07232_b200/csrc`). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError here = header / library mismatch
        fn.restype = res
        fn.argtypes = args
    if lib.bht_sizeof_config() != C.sizeof(Config):
        raise BhtLibraryMissing("bht_config layout mismatch between _lib.py and libbht_b200.so")
    _lib = lib
    return lib


def last_error() -> str:
    return load().bht_last_error_string().decode()
