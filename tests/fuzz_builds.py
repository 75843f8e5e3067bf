"""Randomised parity sweep of the bulk-build schedules (under tests/ because it uses the CPU oracle as its checker; not collected by pytest: run on the GPU box for a few minutes, `python tests/fuzz_builds.py [seed] [seconds]`).
For random (kind, b, load factor, n, schedule, batches): the stored multiset equals the inserted set, every pair is
admissible, finds answer exactly — checked with the CPU oracle reading the GPU's store."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import numpy as np
import torch
import paper_2108_07232_b200 as bht
from oracle import binding

ora = binding.oracle()
rng = np.random.Generator(np.random.MT19937(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 120.0
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()
t0, cases, failed_builds = time.time(), 0, 0
SIZES = [1, 2, 31, 32, 33, 255, 2047, 2048, 2049, 4095, 4097, 10_000, 65_537, 150_001, 400_003, 1_000_003]
while time.time() - t0 < budget:
    kind = rng.choice(["bcht", "bcht", "bcht", "1cht", "bp2ht", "iht"])
    b = 1 if kind == "1cht" else int(rng.choice([1, 2, 4, 8, 16, 32, 64] if kind == "bcht" else [8, 16, 32]))
    lf = float(rng.choice([0.3, 0.5, 0.7, 0.8, 0.9, 0.95] if kind in ("bcht",) and b >= 8 else [0.3, 0.5, 0.6]))
    n = int(rng.choice(SIZES)) + int(rng.integers(0, 3))
    mode = int(rng.choice([0, 1, 2, 3]))
    n_batches = int(rng.choice([1, 1, 2, 3]))
    throttle = bool(rng.integers(0, 2))
    how = str(rng.choice(["bulk", "bulk", "chunked", "host"]))  # bht_insert per batch / one chunked build / host arrays
    raw = np.unique(rng.integers(0, 0xFFFFFFFF, size=2 * n + 64, dtype=np.uint64).astype(np.uint32))
    rng.shuffle(raw)
    keys, absent = raw[:n], raw[n:n + min(n, 5000) + 1]
    vals = rng.integers(0, 0xFFFFFFFF, size=n, dtype=np.uint64).astype(np.uint32)
    try:
        cfg = bht.make_config(kind, n, lf, b, seed=int(rng.integers(0, 2**62)))
    except ValueError:
        continue
    table = bht.HashTable(cfg, 0)
    table.set_blocked_insert(mode)
    table.set_tail_throttle(throttle)
    cuts = sorted(set([0, n] + [int(x) for x in rng.integers(0, n + 1, size=n_batches - 1)]))
    off = int(rng.integers(0, 4))  # unaligned device slices
    inserted = failed = 0
    if how == "chunked":
        table.build_begin(n)
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        if how == "host":
            o = table.insert(keys[lo:hi], vals[lo:hi])
        else:
            dk = dev(np.concatenate([np.zeros(off, np.uint32), keys[lo:hi]]))[off:]
            dv = dev(np.concatenate([np.zeros(off, np.uint32), vals[lo:hi]]))[off:]
            if how == "chunked":
                table.build_feed(dk, dv)
                continue
            o = table.insert(dk, dv)
        inserted += o.inserted
        failed += o.failed
    if how == "chunked":
        o = table.build_end()
        inserted, failed = o.inserted, o.failed
    desc = f"kind={kind} b={b} lf={lf} n={n} mode={mode} batches={cuts} throttle={throttle} off={off} how={how}"
    assert inserted + failed == n, desc
    assert table.occupied_slots() == inserted and table.count_inadmissible() == 0, desc
    store = table.download_store()
    got = table.find(dev(keys)).cpu().numpy().view(np.uint32)
    gota = table.find(dev(absent)).cpu().numpy().view(np.uint32)
    assert np.all(gota == 0xFFFFFFFF), desc
    if failed == 0:
        assert np.array_equal(got, vals), desc
        want = np.sort((vals.astype(np.uint64) << np.uint64(32)) | keys.astype(np.uint64))
        assert np.array_equal(np.sort(store[store != np.uint64(0xFFFFFFFFFFFFFFFF)]), want), desc
        ocfg = binding.Config.from_buffer_copy(bytes(cfg))
        otab = ora.table(ocfg)
        otab.upload_store(store)
        assert otab.check_admissibility() == 0, desc
        w, hits, _ = otab.find_bulk(keys)
        assert hits == n and np.array_equal(w, vals), desc
    else:
        failed_builds += 1
        dropped = np.sort(table.failed_keys())
        assert np.array_equal(np.sort(keys[got == 0xFFFFFFFF]), dropped), desc
    table.close()
    cases += 1
print(f"fuzz ok: {cases} cases in {time.time() - t0:.0f} s ({failed_builds} builds dropped pairs and reported them exactly)")
