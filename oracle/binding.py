"""ctypes bindings of the two CPU checkers — TEST INFRASTRUCTURE ONLY.

* ``Oracle``  -> oracle/liboracle.so        plain-C restatement (oracle/bht_oracle.c)
* ``Ref``     -> oracle/_ref/libbht_ref.so  the unmodified reference + oracle/ref_shim.cpp

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import this module.  The product package (paper_2108_07232_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbht_ref.so")

KINDS = {"1cht": 0, "bcht": 1, "bp2ht": 2, "iht": 3}
EMPTY = 0xFFFFFFFF
EMPTY_SLOT = 0xFFFFFFFFFFFFFFFF


class Config(C.Structure):
    """Same layout as bht_config / or_config / the shim's pod_config."""

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
        ("alpha", C.c_uint64 * 4),
        ("beta", C.c_uint64 * 4),
        ("range", C.c_uint64 * 4),
    ]

    def as_dict(self):
        h = self.n_hashes
        return {
            "kind": self.kind,
            "bucket_size": self.bucket_size,
            "num_buckets": self.num_buckets,
            "capacity": self.capacity,
            "n_hashes": h,
            "threshold": self.threshold,
            "max_chain": self.max_chain,
            "seed": self.seed,
            "alpha": [int(self.alpha[i]) for i in range(h)],
            "beta": [int(self.beta[i]) for i in range(h)],
            "range": [int(self.range[i]) for i in range(h)],
        }

    def copy(self):
        c = Config()
        C.memmove(C.byref(c), C.byref(self), C.sizeof(Config))
        return c


def craft(kind, m, b, hashes, threshold=0, max_chain=8, seed=1):
    """Handcrafted configuration, as proj/tests/test_table.cpp:15-28 (`craft`)."""
    c = Config()
    c.kind = KINDS[kind] if isinstance(kind, str) else kind
    c.num_buckets = m
    c.bucket_size = b
    c.capacity = m * b
    c.n_hashes = len(hashes)
    for i, (a, be, r) in enumerate(hashes):
        c.alpha[i], c.beta[i], c.range[i] = a, be, r
    c.threshold = threshold
    c.max_chain = max_chain
    c.seed = seed
    return c


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _p32(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _p64(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _p8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def build_libs(ref=True):
    """Compiles liboracle.so (always) and oracle/_ref (only where /root/reference exists)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    if ref:
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(self.path)
        self.lib = C.CDLL(self.path)
        L, p = self.lib, self.prefix
        u32, u64, i32, i64, dbl, vp = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double, C.c_void_p
        P32, P64, P8 = C.POINTER(u32), C.POINTER(u64), C.POINTER(C.c_uint8)

        def sig(name, res, *args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = list(args)
            return f

        self._bucket_index = sig("bucket_index", u64, u64, u64, u64, u32)
        self._splitmix64 = sig("splitmix64", u64, u64)
        self._mix_seed = sig("mix_seed", u64, u64, u64)
        self._xorshift_stream = sig("xorshift_stream", None, u64, u64, P64)
        self._next_below_stream = sig("next_below_stream", None, u64, u32, u64, P32)
        self._hash_count = sig("hash_count", u32, i32)
        self._default_max_chain = sig("default_max_chain", u32, u64)
        self._make_config = sig("make_config", C.c_int, i32, u64, dbl, u32, i64, u64, i64, C.POINTER(Config))
        self._pack_pair = sig("pack_pair", u64, u32, u32)
        self._sizeof_config = sig("sizeof_config", C.c_size_t)
        self._value_for_key = sig("value_for_key", u32, u32)
        self._generate_keys = sig("generate_keys", None, u64, u64, P32)
        self._bucket_sectors = sig("bucket_sectors", u32, u32)
        self._predict_sectors = sig("predict_sectors", dbl, i32, u32, dbl, i32)
        self._table_create = sig("table_create", vp, C.POINTER(Config))
        self._table_destroy = sig("table_destroy", None, vp)
        self._table_inserted = sig("table_inserted", u64, vp)
        self._occupied_slots = sig("occupied_slots", u64, vp)
        self._slot_at = sig("slot_at", u64, vp, u64)
        self._poke_slot = sig("poke_slot", None, vp, u64, u64)
        self._download_store = sig("download_store", None, vp, P64)
        self._upload_store = sig("upload_store", None, vp, P64)
        self._find_key = sig("find_key", C.c_int, vp, u32, P32, P64)
        self._find_key_no_early_exit = sig("find_key_no_early_exit", C.c_int, vp, u32, P32)
        self._check_admissibility = sig("check_admissibility", u64, vp)
        self._sig = sig

    # ---- scalar helpers -------------------------------------------------------------------
    def bucket_index(self, alpha, beta, rng, key):
        return int(self._bucket_index(alpha, beta, rng, key))

    def mix_seed(self, seed, stream):
        return int(self._mix_seed(seed, stream))

    def splitmix64(self, x):
        return int(self._splitmix64(x))

    def xorshift_stream(self, seed, n):
        out = np.empty(n, dtype=np.uint64)
        self._xorshift_stream(seed, n, _p64(out))
        return out

    def next_below_stream(self, seed, bound, n):
        out = np.empty(n, dtype=np.uint32)
        self._next_below_stream(seed, bound, n, _p32(out))
        return out

    def hash_count(self, kind):
        return int(self._hash_count(kind))

    def default_max_chain(self, n):
        return int(self._default_max_chain(n))

    def make_config(self, kind, n, lf, b, threshold=None, seed=0, max_chain=None):
        """Returns a Config, or raises ValueError where the reference throws invalid_argument."""
        k = KINDS[kind] if isinstance(kind, str) else kind
        c = Config()
        rc = self._make_config(k, n, lf, b, -1 if threshold is None else threshold, seed,
                               -1 if max_chain is None else max_chain, C.byref(c))
        if rc:
            raise ValueError("make_config: invalid argument")
        return c

    def pack_pair(self, k, v):
        return int(self._pack_pair(k, v))

    def sizeof_config(self):
        return int(self._sizeof_config())

    def value_for_key(self, k):
        return int(self._value_for_key(k))

    def values_for_keys(self, keys):
        keys = _u32(keys)
        v = keys ^ np.uint32(0x5A5A5A5A)
        v[v == EMPTY] &= np.uint32(0x7FFFFFFF)
        return v

    def generate_keys(self, seed, n):
        out = np.empty(n, dtype=np.uint32)
        self._generate_keys(seed, n, _p32(out))
        return out

    def bucket_sectors(self, b):
        return int(self._bucket_sectors(b))

    def predict_sectors(self, kind, b, probes, op):
        k = KINDS[kind] if isinstance(kind, str) else kind
        return float(self._predict_sectors(k, b, probes, {"insert": 0, "find": 1}[op]))

    def bucket_index_many(self, alpha, beta, rng, keys):
        keys = _u32(keys)
        return np.fromiter((self._bucket_index(alpha, beta, rng, int(k)) for k in keys), dtype=np.uint64, count=len(keys))


class _Table:
    def __init__(self, owner, handle, cfg):
        self.o = owner
        self.h = handle
        self.cfg = cfg

    def close(self):
        if self.h:
            self.o._table_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def inserted(self):
        return int(self.o._table_inserted(self.h))

    def occupied_slots(self):
        return int(self.o._occupied_slots(self.h))

    def slot_at(self, i):
        return int(self.o._slot_at(self.h, i))

    def poke_slot(self, i, s):
        self.o._poke_slot(self.h, i, s)

    def download_store(self):
        out = np.empty(self.cfg.capacity, dtype=np.uint64)
        self.o._download_store(self.h, _p64(out))
        return out

    def upload_store(self, store):
        store = np.ascontiguousarray(store, dtype=np.uint64)
        assert store.size == self.cfg.capacity
        self.o._upload_store(self.h, _p64(store))

    def locate(self, key):
        """Global slot index where `key` lives, or -1 (proj/tests/test_table.cpp:31-35)."""
        st = self.download_store()
        idx = np.nonzero((st & np.uint64(0xFFFFFFFF)) == np.uint64(key))[0]
        return int(idx[0]) if idx.size else -1

    def find_key(self, key):
        """-> (found, value, probes)"""
        v = C.c_uint32(0)
        p = C.c_uint64(0)
        r = self.o._find_key(self.h, key, C.byref(v), C.byref(p))
        return bool(r == 1), int(v.value), int(p.value)

    def find_key_no_early_exit(self, key):
        v = C.c_uint32(0)
        r = self.o._find_key_no_early_exit(self.h, key, C.byref(v))
        return bool(r == 1), int(v.value)

    def check_admissibility(self):
        return int(self.o._check_admissibility(self.h))


class OracleTable(_Table):
    def __init__(self, owner, handle, cfg):
        super().__init__(owner, handle, cfg)
        self.rng = C.c_uint64(owner._rng_init(1))

    def seed_rng(self, seed):
        self.rng = C.c_uint64(self.o._rng_init(seed))

    def insert_pair(self, key, value, prose=False):
        """-> (status, probes); status 1 inserted, 0 failed, -1 kind mismatch"""
        p = C.c_uint64(0)
        r = self.o._insert_pair(self.h, key, value, C.byref(self.rng), int(prose), C.byref(p))
        return int(r), int(p.value)

    def build(self, keys, values=None, prose=False):
        """build() sequential (table.cpp:224-238). -> dict(inserted, probes, failed_index)"""
        keys = _u32(keys)
        vals = None if values is None else _u32(values)
        p = C.c_uint64(0)
        fi = C.c_uint64(0)
        r = self.o._build(self.h, _p32(keys), None if vals is None else _p32(vals), len(keys), int(prose),
                          C.byref(p), C.byref(fi))
        if r < 0:
            raise ValueError("build: key set exceeds table capacity")
        return {"inserted": int(r), "probes": int(p.value), "failed_index": int(fi.value),
                "success": int(r) == len(keys)}

    def insert_all(self, keys, values=None, prose=False):
        keys = _u32(keys)
        vals = None if values is None else _u32(values)
        p = C.c_uint64(0)
        flags = np.zeros(len(keys), dtype=np.uint8)
        r = self.o._insert_all(self.h, _p32(keys), None if vals is None else _p32(vals), len(keys), int(prose),
                               C.byref(p), _p8(flags))
        return {"inserted": int(r), "probes": int(p.value), "failed": flags.astype(bool)}

    def find_bulk(self, keys):
        """-> (values[u32] with EMPTY for misses, hits, probes)"""
        keys = _u32(keys)
        out = np.empty(len(keys), dtype=np.uint32)
        p = C.c_uint64(0)
        hits = self.o._find_bulk(self.h, _p32(keys), len(keys), _p32(out), C.byref(p))
        return out, int(hits), int(p.value)


class Oracle(_Lib):
    prefix = "or_"
    path = ORACLE_SO

    def __init__(self):
        super().__init__()
        u32, u64, i32, vp = C.c_uint32, C.c_uint64, C.c_int32, C.c_void_p
        P32, P64, P8 = C.POINTER(u32), C.POINTER(u64), C.POINTER(C.c_uint8)
        sig = self._sig
        self._rng_init = sig("rng_init", u64, u64)
        self._insert_pair = sig("insert_pair", C.c_int, vp, u32, u32, P64, C.c_int, P64)
        self._build = sig("build", C.c_int64, vp, P32, P32, u64, C.c_int, P64, P64)
        self._insert_all = sig("insert_all", C.c_int64, vp, P32, P32, u64, C.c_int, P64, P8)
        self._find_bulk = sig("find_bulk", u64, vp, P32, u64, P32, P64)
        self._mt_stream = sig("mt19937_64_stream", None, u64, u64, P64)
        self._shard_of = sig("shard_of", u32, u64, u64, u32, u32)

    def table(self, cfg):
        h = self._table_create(C.byref(cfg))
        if not h:
            raise ValueError("hash_table: config carries wrong number of hash functions")
        return OracleTable(self, h, cfg.copy())

    def mt19937_64_stream(self, seed, n):
        out = np.empty(n, dtype=np.uint64)
        self._mt_stream(seed, n, _p64(out))
        return out

    def shard_of(self, alpha, beta, n_shards, key):
        return int(self._shard_of(alpha, beta, n_shards, key))


class RefTable(_Table):
    def __init__(self, owner, handle, cfg):
        super().__init__(owner, handle, cfg)
        self._rng = owner._rng_create(1)

    def seed_rng(self, seed):
        self.o._rng_destroy(self._rng)
        self._rng = self.o._rng_create(seed)

    def close(self):
        if getattr(self, "_rng", None):
            self.o._rng_destroy(self._rng)
            self._rng = None
        super().close()

    def insert_pair(self, key, value, prose=False):
        p = C.c_uint64(0)
        r = self.o._insert_pair(self.h, key, value, self._rng, int(prose), C.byref(p))
        return int(r), int(p.value)

    def variant_insert(self, variant, key, value, prose=False):
        p = C.c_uint64(0)
        return int(self.o._variant_insert(self.h, variant, key, value, self._rng, int(prose), C.byref(p))), int(p.value)

    def insert_pairs(self, keys, values=None, prose=False, stop_on_failure=True):
        keys = _u32(keys)
        vals = None if values is None else _u32(values)
        p = C.c_uint64(0)
        flags = np.zeros(len(keys), dtype=np.uint8)
        r = self.o._insert_pairs(self.h, _p32(keys), None if vals is None else _p32(vals), len(keys), int(prose),
                                 int(stop_on_failure), C.byref(p), _p8(flags))
        return {"inserted": int(r), "probes": int(p.value), "failed": flags.astype(bool),
                "success": int(r) == len(keys)}

    def find_bulk(self, keys, threads=1):
        keys = _u32(keys)
        out = np.empty(len(keys), dtype=np.uint32)
        p = C.c_uint64(0)
        ns = C.c_uint64(0)
        hits = self.o._find_bulk(self.h, _p32(keys), len(keys), _p32(out), threads, C.byref(p), C.byref(ns))
        self.last_find_seconds = ns.value * 1e-9
        return out, int(hits), int(p.value)

    def find_bulk_timed(self, keys, threads=1):
        """-> (values, hits, probes, seconds of the find loop alone)"""
        out, hits, probes = self.find_bulk(keys, threads)
        return out, hits, probes, self.last_find_seconds

    def check_membership(self, keys, n_negative, seed):
        keys = _u32(keys)
        out = (C.c_uint64 * 3)()
        self.o._check_membership(self.h, _p32(keys), len(keys), n_negative, seed, out)
        return {"false_negatives": int(out[0]), "wrong_values": int(out[1]), "false_positives": int(out[2])}


class Ref(_Lib):
    prefix = "ref_"
    path = REF_SO

    def __init__(self):
        super().__init__()
        u32, u64, i32, vp = C.c_uint32, C.c_uint64, C.c_int32, C.c_void_p
        P32, P64, P8 = C.POINTER(u32), C.POINTER(u64), C.POINTER(C.c_uint8)
        sig = self._sig
        self._rng_create = sig("rng_create", vp, u64)
        self._rng_destroy = sig("rng_destroy", None, vp)
        self._insert_pair = sig("insert_pair", C.c_int, vp, u32, u32, vp, C.c_int, P64)
        self._variant_insert = sig("variant_insert", C.c_int, vp, C.c_int, u32, u32, vp, C.c_int, P64)
        self._insert_pairs = sig("insert_pairs", C.c_int64, vp, P32, P32, u64, C.c_int, C.c_int, P64, P8)
        self._build = sig("build", vp, P32, u64, C.POINTER(Config), C.c_int, C.c_uint, C.c_int, P64)
        self._find_bulk = sig("find_bulk", u64, vp, P32, u64, P32, C.c_uint, P64, P64)
        self._check_membership = sig("check_membership", None, vp, P32, u64, u64, u64, P64)
        self._generate_queries = sig("generate_queries", C.c_int, P32, u64, C.c_double, u64, u64, P32, P32, P8)
        self._hardware_concurrency = sig("hardware_concurrency", C.c_uint)
        self._core_is_reference = sig("core_is_reference", C.c_int)
        self._has_experiments = sig("has_experiments", C.c_int)
        if self._has_experiments():
            dbl, P_D, cp = C.c_double, C.POINTER(C.c_double), C.c_char_p
            self._config_to_json = sig("config_to_json", C.c_size_t, C.POINTER(Config), cp, C.c_size_t)
            self._config_from_json = sig("config_from_json", C.c_int, cp, C.POINTER(Config))
            self._spec_roundtrip = sig("spec_roundtrip", C.c_size_t, cp, cp, C.c_size_t)
            self._run_experiment = sig("run_experiment", C.c_size_t, cp, C.c_int, cp, C.c_size_t)
            self._run_trial = sig("run_trial", C.c_int, i32, u32, u32, u64, dbl, P_D, u32, C.c_uint, C.c_uint, u64, P_D)
            self._run_success_rate = sig("run_success_rate", C.c_int, i32, u32, u32, u64, P_D, u32, C.c_uint, u64, P32)

    # ---- experiment protocol / wire formats (experiments.cpp, core.cpp:70-109) ----
    def has_experiments(self):
        return bool(self._has_experiments())

    def _text(self, fn, *args):
        buf = C.create_string_buffer(1 << 20)
        n = fn(*args, buf, len(buf))
        if n == 0:
            raise ValueError("reference threw")
        return buf.value.decode()

    def config_to_json(self, cfg):
        return self._text(self._config_to_json, C.byref(cfg))

    def config_from_json(self, text):
        cfg = Config()
        if self._config_from_json(text.encode(), C.byref(cfg)):
            raise ValueError("config_from_json: invalid")
        return cfg

    def spec_roundtrip(self, text):
        return self._text(self._spec_roundtrip, text.encode())

    def run_experiment(self, spec_json, fmt="csv"):
        return self._text(self._run_experiment, spec_json.encode(), 0 if fmt == "csv" else 1)

    def run_trial(self, kind, b, threshold_pct, n, lf, ratios, trials, max_failures, seed):
        r = (C.c_double * max(1, len(ratios)))(*ratios)
        out = (C.c_double * (5 + len(ratios)))()
        if self._run_trial(kind, b, threshold_pct, n, lf, r, len(ratios), trials, max_failures, seed, out):
            raise ValueError("run_trial: reference threw")
        return {"successes": int(out[0]), "failures": int(out[1]), "budget_exhausted": bool(out[2]), "realized_lf": out[3],
                "insert_mean_probes": out[4], "find_mean_probes": [out[5 + i] for i in range(len(ratios))]}

    def run_success_rate(self, kind, b, threshold_pct, n, lf_grid, success_trials, seed):
        g = (C.c_double * len(lf_grid))(*lf_grid)
        succ = (C.c_uint32 * len(lf_grid))()
        if self._run_success_rate(kind, b, threshold_pct, n, g, len(lf_grid), success_trials, seed, succ):
            raise ValueError("run_success_rate: reference threw")
        return [int(x) for x in succ]

    def core_is_reference(self):
        return bool(self._core_is_reference())

    def hardware_concurrency(self):
        return int(self._hardware_concurrency())

    def table(self, cfg):
        h = self._table_create(C.byref(cfg))
        if not h:
            raise ValueError("hash_table: config carries wrong number of hash functions")
        return RefTable(self, h, cfg.copy())

    def build(self, keys, cfg, parallel=False, workers=0, prose=False):
        """The reference's own build() (value_for_key values). -> (RefTable, outcome dict)"""
        keys = _u32(keys)
        out = (C.c_uint64 * 5)()
        h = self._build(_p32(keys), len(keys), C.byref(cfg), int(parallel), workers, int(prose), out)
        if not h:
            raise ValueError("build: key set exceeds table capacity")
        failed = None if out[2] == EMPTY_SLOT else int(out[2])
        return RefTable(self, h, cfg.copy()), {"success": bool(out[0]), "inserted": int(out[1]), "failed_key": failed,
                                               "probes": int(out[3]), "seconds": out[4] * 1e-9}

    def generate_queries(self, keys, ratio, q, seed):
        """-> (query keys, expected values (EMPTY for negatives), present flags)"""
        keys = _u32(keys)
        qk = np.empty(q, dtype=np.uint32)
        ev = np.empty(q, dtype=np.uint32)
        pr = np.empty(q, dtype=np.uint8)
        if self._generate_queries(_p32(keys), len(keys), ratio, q, seed, _p32(qk), _p32(ev), _p8(pr)):
            raise ValueError("generate_queries: invalid argument")
        return qk, ev, pr.astype(bool)


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build_libs(ref=False)
        _oracle = Oracle()
    return _oracle


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref
