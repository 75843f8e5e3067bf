"""bht-b200: bulk build / bulk find for BCHT, BP2HT, IHT and 1CHT on B200 (sm_100a).

The package is the host-side mirror of the reference table API over the C ABI in include/bht_b200.h.
Importing it loads lib/libbht_b200.so and fails loudly if that library has not been built: there is no
CPU fallback on any product path.
"""
from . import _lib

_lib.load()

from .table import (  # noqa: E402
    EMPTY_KEY, EMPTY_SLOT, EMPTY_VALUE, KINDS, OP_FIND, OP_INSERT, BuildOutcome, CapacityError, CudaError, FindStats,
    HashTable, KindMismatchError, bucket_index, build, craft_config, default_max_chain, generate_unique_keys,
    hash_count, hash_keys, hash_table, kernel_launch_count, make_config, mix_seed, pack_pair, predict_sectors,
    reload_tuning, unpack_slot, value_for_key, values_for_keys,
)
from ._lib import Config  # noqa: E402
from . import experiments, workload  # noqa: E402,F401
from .sharded import ShardedTable, LocalShardedTable, CudaShardOps, RoutingOverflow, shard_constants  # noqa: E402

__all__ = [n for n in dir() if not n.startswith("_")]
