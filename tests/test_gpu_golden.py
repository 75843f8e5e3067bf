"""The committed fixtures of the UNMODIFIED reference (tests/golden/reference_vectors.npz) against the CUDA path."""
import os

import numpy as np
import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
EMPTY = 0xFFFFFFFF


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_vectors.npz"))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint32)


def cfg_from_row(bht, row):
    c = bht.Config()
    c.kind, c.bucket_size, c.num_buckets, c.capacity = int(row[0]), int(row[1]), int(row[2]), int(row[3])
    c.n_hashes, c.threshold, c.max_chain, c.seed = int(row[4]), int(row[5]), int(row[6]), int(row[7])
    for i in range(4):
        c.alpha[i], c.beta[i], c.range[i] = int(row[8 + i]), int(row[12 + i]), int(row[16 + i])
    return c


def test_golden_hash_vectors_on_device(bht, gold):
    a, b, r, k, want = (gold[x] for x in ("hash_alpha", "hash_beta", "hash_range", "hash_key", "hash_out"))
    for i in range(0, 256):  # one launch per (alpha, beta, range) tuple
        got = host(bht.hash_keys(int(a[i]), int(b[i]), int(r[i]), dev(k[i:i + 1])))
        assert int(got[0]) == int(want[i])
    # one long launch with fixed constants against numpy's u64 arithmetic of hash.hpp:21-23
    keys = k.astype(np.uint64)
    got = host(bht.hash_keys(int(a[7]), int(b[7]), int(r[7]), dev(k))).astype(np.uint64)
    assert np.array_equal(got, ((a[7] * keys + b[7]) % np.uint64(4294967291)) % r[7])


def test_golden_tables_find_on_reference_layout(bht, gold):
    """Upload the reference-built store: answers and probe counts equal the reference's find loop bit for bit."""
    for name in gold["table_cases"]:
        g = lambda f: gold[f"t_{name}_{f}"]  # noqa: E731
        cfg = cfg_from_row(bht, g("cfg"))
        table = bht.HashTable(cfg, 0)
        table.upload_store(g("store"))
        n = g("keys").size
        assert table.inserted() == n
        q = np.concatenate([g("keys"), g("absent")])
        got, st = table.find(dev(q), want_stats=True)
        assert np.array_equal(host(got), g("find_out")), name
        assert st.probes == int(g("find_probes")), name
        assert st.hits == n
        assert np.array_equal(host(table.find_exhaustive(dev(q))), g("find_exhaustive")), name
        assert table.count_inadmissible() == 0
        # and via the host-memory path
        assert np.array_equal(table.find(q), g("find_out")), name


def test_golden_tables_gpu_build(bht, gold):
    """GPU bulk build of the fixture's pairs: same answers as the reference for the same queries; stored multiset
    equals the reference's stored multiset (layout may differ)."""
    for name in gold["table_cases"]:
        g = lambda f: gold[f"t_{name}_{f}"]  # noqa: E731
        cfg = cfg_from_row(bht, g("cfg"))
        table, o = bht.build(dev(g("keys")), cfg, dev(g("values")), device=0)
        assert o.success, name
        q = np.concatenate([g("keys"), g("absent")])
        assert np.array_equal(host(table.find(dev(q))), g("find_out")), name
        ref_store = g("store")
        mine = table.download_store()
        full = np.uint64(0xFFFFFFFFFFFFFFFF)
        assert np.array_equal(np.sort(mine[mine != full]), np.sort(ref_store[ref_store != full])), name
        assert table.count_inadmissible() == 0


def test_golden_failed_build_cell(bht, gold):
    cfg = cfg_from_row(bht, gold["fail_cfg"])
    keys = gold["fail_keys"]
    table, o = bht.build(dev(keys), cfg, device=0)
    assert not o.success  # the reference fails on this cell too (bp2ht b=8 at load 1.0)
    dropped = table.failed_keys()
    got = host(table.find(dev(keys)))
    assert np.all(got[np.isin(keys, dropped)] == EMPTY)
    assert np.all(got[~np.isin(keys, dropped)] != EMPTY)
