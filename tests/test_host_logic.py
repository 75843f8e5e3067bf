"""CPU-side checks of the product's host layer: the C-ABI library loads and exports every symbol that
include/bht_b200.h declares, and the host-only entry points (make_config, the division-free hash twin, the
sector model, shard routing, the key bijection) agree bit for bit with the oracle.  No compute call is made."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import binding

P = 4294967291


def header_symbols():
    text = open(os.path.join(ROOT, "include", "bht_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bht_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(bht):
    from paper_2108_07232_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/bht_b200.h but not exported"
    # and the ctypes table covers exactly the header
    assert sorted(_lib.SIGNATURES) == syms


def test_struct_layouts(bht, ora):
    from paper_2108_07232_b200 import _lib
    assert _lib.load().bht_sizeof_config() == C.sizeof(_lib.Config) == ora.sizeof_config() == C.sizeof(binding.Config)
    assert _lib.load().bht_version_string().decode().startswith("bht_b200")


def test_make_config_bit_exact(bht, ora):
    rng = np.random.default_rng(5)
    for kind, b, t in [("bcht", 16, None), ("bcht", 1, None), ("bcht", 64, None), ("1cht", 1, None), ("bp2ht", 8, None),
                       ("bp2ht", 32, None), ("iht", 16, None), ("iht", 16, 3), ("iht", 32, 32), ("iht", 2, None)]:
        for _ in range(20):
            n = int(rng.integers(1, 600_000_000))
            lf = float(rng.uniform(0.05, 1.0))
            seed = int(rng.integers(0, 1 << 63))
            mc = None if rng.random() < 0.5 else int(rng.integers(0, 1000))
            if kind == "iht" and b == 2 and t is None:
                with pytest.raises(ValueError):  # default threshold 2*80/100 = 1 is fine; b=1 would give 0
                    bht.make_config("iht", n, lf, 1, seed=seed)
            a = bht.make_config(kind, n, lf, b, threshold=t, seed=seed, max_chain=mc)
            o = ora.make_config(kind, n, lf, b, threshold=t, seed=seed, max_chain=mc)
            assert bytes(a) == bytes(o), (kind, n, lf, b, t, seed)
    for n in [1, 2, 3, 4, 5, 1000, 100_000, 1_000_000, 50_000_000, 1 << 32, (1 << 40) + 1]:
        assert bht.default_max_chain(n) == ora.default_max_chain(n)
    for k in range(4):
        assert bht.hash_count(k) == ora.hash_count(k) == [4, 3, 2, 3][k]


def test_make_config_rejections(bht):
    # proj/tests/test_core.cpp:47-65 -> std::invalid_argument
    for bad in [("bcht", 0, 0.5, 16), ("bcht", 10, 0.0, 16), ("bcht", 10, -1.0, 16), ("bcht", 10, 1.0001, 16),
                ("bcht", 10, float("nan"), 16), ("bcht", 10, 0.5, 0), ("bcht", 10, 0.5, 12), ("bcht", 10, 0.5, 128),
                ("1cht", 10, 0.5, 2)]:
        with pytest.raises(ValueError):
            bht.make_config(*bad)
    with pytest.raises(ValueError):
        bht.make_config("iht", 10, 0.5, 16, threshold=17)
    with pytest.raises(ValueError):
        bht.make_config("iht", 10, 0.5, 16, threshold=0)
    with pytest.raises(ValueError):
        bht.make_config("cuckoo", 10, 0.5, 16)
    assert bht.make_config("iht", 1000, 0.8, 16).threshold == 12
    assert bht.make_config("bp2ht", 1000, 0.8, 32).num_buckets == 40


def test_hash_twin_bit_exact(bht, ora):
    """The division-free arithmetic of the device hash stage (host twin) == ((a*k+b) % p) % L (hash.hpp:21-23)."""
    assert bht.bucket_index(1, 0, 10, 7) == 7
    assert bht.bucket_index(3, 4, 3, 7) == 1
    assert bht.bucket_index(2, 0, 5, 4294967290) == 4
    rng = np.random.default_rng(11)
    edge_a = [1, 2, P - 1, P - 2, 0xFFFFFFFA, 1 << 31]
    edge_b = [0, 1, P - 1, 5, 0xFFFFFFFA]
    edge_r = [1, 2, 3, 5, (1 << 32) - 1, P, P - 1, 1 << 31, 3472223, 62_500_000, 34_722_223]
    edge_k = [0, 1, 2, 0xFFFFFFFE, 0xFFFFFFFF, 0x80000000, 0x7FFFFFFF, P, P - 1, 5, 4]
    for a in edge_a:
        for b in edge_b:
            for r in edge_r:
                for k in edge_k:
                    assert bht.bucket_index(a, b, r, k) == ((a * k + b) % P) % r == ora.bucket_index(a, b, r, k)
    for _ in range(50_000):
        a, b = int(rng.integers(1, P)), int(rng.integers(0, P))
        r, k = int(rng.integers(1, 1 << 32)), int(rng.integers(0, 1 << 32))
        assert bht.bucket_index(a, b, r, k) == ((a * k + b) % P) % r
    with pytest.raises(ValueError):
        bht.bucket_index(1 << 32, 0, 5, 1)
    with pytest.raises(ValueError):
        bht.bucket_index(1, 0, 0, 1)


def test_golden_hash_through_host_twin(bht):
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_vectors.npz"))
    for a, b, r, k, want in zip(g["hash_alpha"], g["hash_beta"], g["hash_range"], g["hash_key"], g["hash_out"]):
        assert bht.bucket_index(int(a), int(b), int(r), int(k)) == int(want)


def test_scalar_helpers(bht, ora):
    for s, st in [(0, 0), (1, 0x68617368), (12345, 0x65766963), ((1 << 64) - 1, 7)]:
        assert bht.mix_seed(s, st) == ora.mix_seed(s, st)
    for k in [0, 1, 0x5A5A5A5A, 0xA5A5A5A5, 0xFFFFFFFE, 123456789]:
        assert bht.value_for_key(k) == ora.value_for_key(k)
    ks = np.array([0, 0xA5A5A5A5, 77, 0xFFFFFFFE], dtype=np.uint32)
    assert np.array_equal(bht.values_for_keys(ks), ora.values_for_keys(ks))
    for kind, b, pr in [("bcht", 16, 1.1085), ("bcht", 32, 1.05), ("1cht", 1, 2.7538), ("bp2ht", 16, 2.0), ("iht", 8, 1.48)]:
        assert bht.predict_sectors(kind, b, pr, bht.OP_INSERT) == ora.predict_sectors(kind, b, pr, "insert")
        assert bht.predict_sectors(kind, b, pr, bht.OP_FIND) == ora.predict_sectors(kind, b, pr, "find")
    assert bht.pack_pair(0x11223344, 0xAABBCCDD) == ora.pack_pair(0x11223344, 0xAABBCCDD)
    assert bht.unpack_slot(bht.pack_pair(5, 9)) == (5, 9)
    assert bht.pack_pair(bht.EMPTY_KEY, bht.EMPTY_VALUE) == bht.EMPTY_SLOT


def test_shard_routing_host(bht, ora):
    from paper_2108_07232_b200 import _lib
    lib = _lib.load()
    a, b = bht.shard_constants(1)
    assert 1 <= a < P and 0 <= b < P
    assert bht.shard_constants(1) == (a, b) and bht.shard_constants(2) != (a, b)
    rng = np.random.default_rng(3)
    counts = np.zeros(8, dtype=np.int64)
    for k in rng.integers(0, 1 << 32, size=40_000):
        k = int(k)
        s = lib.bht_shard_of_host(a, b, 8, k)
        assert s == ((((a * k + b) % P) * 8) >> 32) == ora.shard_of(a, b, 8, k)
        counts[s] += 1
    assert counts.min() > 4500 and counts.max() < 5500  # uniform over shards
    assert lib.bht_shard_of_host(a, b, 1, 12345) == 0


def test_unique_key_bijection_host(bht):
    """bht_generate_unique_keys' generator: injective, sentinel-free, seed-dependent (keygen.cpp:50-64 contract)."""
    from paper_2108_07232_b200 import _lib
    lib = _lib.load()
    for seed in [0, 1, 0xDEADBEEFCAFEF00D]:
        ks = np.array([lib.bht_unique_key_host(seed, c) for c in range(20_000)], dtype=np.uint32)
        assert np.unique(ks).size == ks.size and not np.any(ks == 0xFFFFFFFF)
        tail = [lib.bht_unique_key_host(seed, c) for c in range(0xFFFFFFFE - 50, 0xFFFFFFFF)]
        assert 0xFFFFFFFF not in tail and len(set(tail)) == len(tail)
        vs = [lib.bht_synthetic_value_host(seed, int(k)) for k in ks[:2000]]
        assert 0xFFFFFFFF not in vs
    # numpy restatement of mix32 (csrc/hash_stage.cuh) over a full 2^20 window: still injective
    def mix32(k0, k1, x):
        x = x.astype(np.uint32) ^ np.uint32(k0)
        x ^= x >> np.uint32(16)
        x = (x.astype(np.uint64) * 0x85EBCA6B & 0xFFFFFFFF).astype(np.uint32)
        x ^= x >> np.uint32(13)
        x = ((x.astype(np.uint64) + k1) & 0xFFFFFFFF).astype(np.uint32)
        x = (x.astype(np.uint64) * 0xC2B2AE35 & 0xFFFFFFFF).astype(np.uint32)
        x ^= x >> np.uint32(16)
        return x
    seed = 0x1234567899887766
    c = np.arange(1 << 20, dtype=np.uint32)
    y = mix32(seed & 0xFFFFFFFF, seed >> 32, c)
    assert np.unique(y).size == y.size
    assert [int(v) for v in y[:64]] == [lib.bht_unique_key_host(seed, i) if y[i] != 0xFFFFFFFF else None for i in range(64)]


def test_create_without_device_fails_loudly(bht):
    """No CPU fallback: on a box without a GPU bht_create reports a CUDA error instead of computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bht.CudaError):
        bht.HashTable(bht.make_config("bcht", 100, 0.5, 16, seed=1), 0)
    with pytest.raises(ValueError):  # config validation happens before any device work
        bad = bht.make_config("bcht", 100, 0.5, 16, seed=1)
        bad.n_hashes = 2
        bht.HashTable(bad, 0)


def test_product_never_imports_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_2108_07232_b200")
    for dirpath, _dirs, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp", ".cpp")) or f == "Makefile":
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.lower() or all(
                    "import" not in line and "#include" not in line and "liboracle" not in line and "libbht_ref" not in line
                    for line in text.splitlines() if "oracle" in line.lower()), os.path.join(dirpath, f)
    for f in os.listdir(os.path.join(ROOT, "include")):
        assert "oracle/" not in open(os.path.join(ROOT, "include", f)).read()
    for f in os.listdir(os.path.join(ROOT, "tools")):  # measurement scripts run the product, never the checker
        path = os.path.join(ROOT, "tools", f)
        if os.path.isfile(path) and f.endswith(".py"):
            assert "from oracle" not in open(path).read() and "import oracle" not in open(path).read(), path


def test_shard_constants_same_in_c_and_python(bht):
    """bht_shard_constants (csrc/sharded.cu) and sharded.shard_constants derive the routing hash of the sharded table
    the same way, so the single-process handle and the one-rank-per-GPU table build the same shards."""
    lib = bht._lib.load()
    rng = np.random.default_rng(11)
    for seed in [0, 1, 2, 0x73686172, (1 << 64) - 1] + [int(x) for x in rng.integers(0, 1 << 63, size=50)]:
        a, b = C.c_uint64(), C.c_uint64()
        lib.bht_shard_constants(seed, C.byref(a), C.byref(b))
        assert (a.value, b.value) == tuple(bht.shard_constants(seed))
        assert 1 <= a.value < 4294967291 and b.value < 4294967291


def test_bench_reference_arm_contract(ref):
    """`bench.py --impl reference` (the arm the driver runs beside the CUDA one): ONE JSON line on stdout with the
    contract's keys, the reference's own CPU path timed on this host's cores, no GPU needed.  A small key count keeps
    it to seconds; --config names any BASELINE.json cell."""
    import json
    import subprocess
    import sys
    for extra in ([], ["--config", "bp2ht08"]):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
                            "--keys", "300000", "--workload", "numpy"] + extra, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
        assert len(lines) == 1, r.stdout
        line = json.loads(lines[0])
        for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                    "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
            assert key in line, key
        assert line["impl"] == "reference" and line["unit"] == "MKeys/s" and line["value"] > 0
        assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
        assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
        if extra:
            assert "BP2HT" in line["metric"] and line["config"]["kind"] == "bp2ht"


def test_bench_configs_cover_baseline_json():
    """Every configuration BASELINE.json names is a `--config` of bench.py."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    cells = set(bench.CONFIGS.values())
    for want in [("bcht", 16, 0.8, None), ("bcht", 16, 0.9, None), ("bcht", 16, 0.99, None), ("1cht", 1, 0.8, None),
                 ("1cht", 1, 0.9, None), ("bp2ht", 16, 0.6, None), ("bp2ht", 16, 0.99, None), ("iht", 16, 0.9, 12),
                 ("iht", 16, 0.99, 12)]:
        assert want in cells, want
    bench.select_config("iht:32:0.9:25")
    assert (bench.KIND, bench.B, bench.LF, bench.THRESHOLD) == ("iht", 32, 0.9, 25) and "IHT b=32, t=25" in bench.METRIC
    bench.select_config("headline")
    assert bench.METRIC == "insert & find MKeys/s, BCHT b=16, 50M keys, LF 0.9" and bench.HEADLINE
