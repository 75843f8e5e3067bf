"""The reference's own acceptance criteria 1-7 (proj/tests/acceptance.cpp:81-240: the paper's hardware-independent
figures) run against the GPU tables through the host mirror of the reference's trial protocol — same key / hash /
query seeds, same desk scale (n = 10^6; 10^5 for the success-rate sweep of criterion 6), same targets and tolerances.
Success-rate sweeps use 50 builds per load factor instead of 200 to keep the tier within a minute or two (the 99 %
threshold then means 50 of 50)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DESK_N = 1_000_000


@pytest.fixture(scope="module")
def ex():
    from paper_2108_07232_b200 import experiments
    return experiments


def probe_cell(ex, kind, b, tpct, n, lf, ratios, seed, trials=10, max_failures=50):
    """probe_cell (acceptance.cpp:59-71)."""
    return ex.run_trial(ex.TrialCell(ex.KindParams(kind, b, tpct), n=n, lf=lf, positive_ratios=list(ratios), trials=trials,
                                     max_failures=max_failures, seed=seed))


def grid(lo, hi, step=0.01):
    return [round(lo + i * step, 10) for i in range(int(round((hi - lo) / step)) + 1)]


def within(x, target, tol):
    return abs(x - target) <= tol


def test_criterion_1_bcht_insertion_probes_at_lf_099(ex):
    out = probe_cell(ex, "bcht", 16, 0, DESK_N, 0.99, [], 101)
    assert not out.budget_exhausted, out.failures
    assert within(out.insert_mean_probes, 1.43, 0.10), out.insert_mean_probes


def test_criterion_2_bcht_query_probes_at_high_load(ex):
    neg = probe_cell(ex, "bcht", 16, 0, DESK_N, 0.99, [0.0], 102)
    assert not neg.budget_exhausted and within(neg.find_mean_probes[0], 2.8, 0.15), neg
    pos = probe_cell(ex, "bcht", 16, 0, DESK_N, 0.98, [1.0], 103)
    assert not pos.budget_exhausted and pos.find_mean_probes[0] <= 1.5, pos


@pytest.mark.parametrize("kind,b,target,tol", [("1cht", 1, 2.75, 0.15), ("bcht", 8, 1.23, 0.10), ("bcht", 16, 1.11, 0.08),
                                               ("bcht", 32, 1.05, 0.05)])
def test_criterion_3_insertion_probes_by_bucket_size(ex, kind, b, target, tol):
    out = probe_cell(ex, kind, b, 0, DESK_N, 0.9, [], 104 + b)
    assert not out.budget_exhausted and within(out.insert_mean_probes, target, tol), out


def test_criterion_4_bp2ht_probe_counts(bht, ex):
    from paper_2108_07232_b200 import workload
    keys = workload.generate_keys(105, DESK_N, device=0)
    cfg = bht.make_config("bp2ht", DESK_N, 0.8, 32, seed=105)
    table, outcome = bht.build(keys.keys.view(torch.int32), cfg, device=0)
    assert outcome.success
    assert outcome.probes == 2 * outcome.attempted           # insert probes exactly 2.0
    neg = workload.generate_queries(keys, 0.0, DESK_N, 106, device=0)
    _, st = table.find(torch.from_numpy(neg.keys.view(np.int32)).cuda(), want_stats=True, as_kind="bp2ht")
    assert st.hits == 0 and st.probes == 2 * DESK_N            # all-negative probes exactly 2.0
    peak = probe_cell(ex, "bp2ht", 32, 0, DESK_N, 0.92, [1.0, 0.5], 107)
    assert not peak.budget_exhausted, peak.failures
    assert within(peak.find_mean_probes[0], 1.33, 0.05) and within(peak.find_mean_probes[1], 1.67, 0.05), peak


@pytest.mark.parametrize("i,pct,insert_target,positive_target", [(0, 20, 2.68, 2.11), (1, 40, 2.29, 1.86), (2, 60, 1.89, 1.60),
                                                                 (3, 80, 1.49, 1.33)])
def test_criterion_5_iht_probes_across_thresholds(ex, i, pct, insert_target, positive_target):
    out = probe_cell(ex, "iht", 16, pct, DESK_N, 0.86, [1.0], 108 + i)
    assert not out.budget_exhausted, out.failures
    assert within(out.insert_mean_probes, insert_target, 0.15), out.insert_mean_probes
    assert within(out.find_mean_probes[0], positive_target, 0.15), out.find_mean_probes


def test_criterion_5_iht_negative_queries_read_all_three_buckets(bht):
    from paper_2108_07232_b200 import workload
    keys = workload.generate_keys(112, DESK_N, device=0)
    cfg = bht.make_config("iht", DESK_N, 0.86, 16, threshold=12, seed=112)
    for attempt in range(8):
        table, outcome = bht.build(keys.keys.view(torch.int32), cfg, device=0)
        if outcome.success:
            break
        cfg = bht.make_config("iht", DESK_N, 0.86, 16, threshold=12, seed=bht.mix_seed(112, attempt))
    assert outcome.success
    neg = workload.generate_queries(keys, 0.0, DESK_N, 113, device=0)
    _, st = table.find(torch.from_numpy(neg.keys.view(np.int32)).cuda(), want_stats=True, as_kind="iht")
    assert st.hits == 0 and st.probes == 3 * DESK_N


def max_lf(ex, kind, b, tpct, n, lo, hi, trials, seed):
    sr = ex.run_success_rate(ex.KindParams(kind, b, tpct), n, grid(lo, hi), trials, seed)
    return sr.max_load_factor or 0.0, sr


def test_criterion_6_achievable_load_factors(ex):
    n, trials = 100_000, 50
    bcht, _ = max_lf(ex, "bcht", 16, 0, n, 0.93, 0.99, trials, 114)
    iht, _ = max_lf(ex, "iht", 32, 80, n, 0.86, 0.96, trials, 114)
    bp2ht, _ = max_lf(ex, "bp2ht", 32, 0, n, 0.86, 0.96, trials, 114)
    one, _ = max_lf(ex, "1cht", 1, 0, n, 0.80, 0.93, trials, 114)
    assert bcht >= 0.97 and iht >= 0.90 and bp2ht >= 0.90 and one >= 0.86, (bcht, iht, bp2ht, one)
    assert bcht > iht and bcht > bp2ht and iht > one and bp2ht > one, (bcht, iht, bp2ht, one)


@pytest.mark.parametrize("kind,tpct,b,target,lo,hi", [("bp2ht", 0, 8, 0.65, 0.61, 0.71), ("bp2ht", 0, 16, 0.84, 0.80, 0.90),
                                                      ("bp2ht", 0, 32, 0.92, 0.88, 0.96), ("iht", 80, 8, 0.70, 0.66, 0.76),
                                                      ("iht", 80, 16, 0.86, 0.82, 0.92), ("iht", 80, 32, 0.93, 0.89, 0.97)])
def test_criterion_7_peak_loads_of_the_stable_tables(ex, kind, tpct, b, target, lo, hi):
    got, sr = max_lf(ex, kind, b, tpct, DESK_N, lo, hi, 50, 115)
    if not within(got, target, 0.03):
        # 50 of 50 is a noisier (and upward-biased) estimate of ">= 99 %" than the reference's 198 of 200: a borderline
        # figure is settled with the reference's own 200 builds per load factor (acceptance.cpp:214-240)
        got, sr = max_lf(ex, kind, b, tpct, DESK_N, lo, hi, 200, 115)
    assert within(got, target, 0.03), (got, [(p.lf, p.successes) for p in sr.points])


# ---- criteria 8-10: the reference's OWN checkers (check_membership, check_admissibility, oracle.cpp:13-54) run on GPU-built
# ---- stores handed over in the reference's dump layout --------------------------------------------------------------

def safe_lf(kind, b):
    """acceptance.cpp:257-265."""
    return {"1cht": 0.80, "bcht": 0.95, "bp2ht": 0.88 if b >= 32 else (0.80 if b == 16 else 0.60),
            "iht": 0.88 if b >= 32 else (0.82 if b == 16 else 0.62)}[kind]


def correctness_suite(ref, cfg, table, keys_host, seed):
    """correctness_suite (acceptance.cpp:267-281): membership {false negatives, wrong values, false positives} over the
    keys and as many guaranteed-absent keys, and admissibility, by the reference's code on the GPU table's store."""
    from conftest import to_oracle_cfg
    rt = ref.table(to_oracle_cfg(cfg))
    try:
        rt.upload_store(table.download_store())
        report = rt.check_membership(keys_host, len(keys_host), seed)
        return report == {"false_negatives": 0, "wrong_values": 0, "false_positives": 0} and rt.check_admissibility() == 0
    finally:
        rt.close()


def test_criterion_8_randomized_correctness_properties(bht, ex, ref, ora):
    """acceptance.cpp:283-368: 100 random (kind, b, n, load factor, threshold) configurations drawn from mt19937_64(116) as
    the reference draws them, built in bulk on the GPU (builds alternate caller order / blocked schedules where the
    reference alternates sequential / 8 workers), all clean; then the early-exit differential on 10^6 mixed queries."""
    from paper_2108_07232_b200 import workload
    stream = iter(ora.mt19937_64_stream(116, 4000).tolist())
    kinds = ["1cht", "bcht", "bp2ht", "iht"]  # table_kind order (core.hpp:43)
    sizes = [8, 16, 32]
    configs = clean = 0
    while configs < 100:
        kind = kinds[next(stream) % 4]
        b = 1 if kind == "1cht" else sizes[next(stream) % 3]
        n = 2000 + next(stream) % 50000
        lf = 0.30 + (safe_lf(kind, b) - 0.30) * ((next(stream) % 1000) / 999.0)
        tpct = 20 + 20 * (next(stream) % 4)
        parallel = configs % 2 == 1
        configs += 1
        keys = workload.generate_keys(next(stream), n, device=0)
        threshold = max(1, b * tpct // 100) if kind == "iht" else None
        cfg = bht.make_config(kind, n, lf, b, threshold=threshold, seed=next(stream))
        table = bht.HashTable(cfg, 0)
        table.set_blocked_insert(3 if parallel else 0)
        d_keys = keys.keys.view(torch.int32)
        outcome = table.insert(d_keys, bht.values_for_keys(d_keys))
        assert outcome.success, (kind, b, lf, n)   # every configuration is at or below its variant's safe load factor
        clean += correctness_suite(ref, cfg, table, keys.keys.cpu().numpy(), next(stream))
        table.close()
    assert clean == configs == 100
    keys = workload.generate_keys(117, DESK_N, device=0)
    d_keys = keys.keys.view(torch.int32)
    for attempt in range(20):
        cfg = bht.make_config("bcht", DESK_N, 0.98, 16, seed=117 if attempt == 0 else 118 + attempt)
        table, outcome = bht.build(d_keys, cfg, device=0)
        if outcome.success:
            break
    assert outcome.success
    q = torch.from_numpy(workload.generate_queries(keys, 0.5, DESK_N, 119, device=0).keys.view(np.int32)).cuda()
    assert torch.equal(table.find(q, as_kind="bcht"), table.find_exhaustive(q))


@pytest.mark.parametrize("kind,b,threshold", [("1cht", 1, None), ("bcht", 16, None), ("bp2ht", 32, None), ("iht", 32, 25)])
def test_criterion_9_concurrent_builds(bht, ref, kind, b, threshold):
    """acceptance.cpp:371-423: a concurrent build of 10^6 keys at LF 0.8 is clean under the reference's checkers; for the
    stable tables, pairs recorded right after their own batch never move while seven more batches are inserted."""
    from paper_2108_07232_b200 import workload
    keys = workload.generate_keys(120 + b, DESK_N, device=0)
    cfg = bht.make_config(kind, DESK_N, 0.8, b, threshold=threshold, seed=120 + b)
    d_keys = keys.keys.view(torch.int32)
    table, outcome = bht.build(d_keys, cfg, device=0)
    assert outcome.success
    assert correctness_suite(ref, cfg, table, keys.keys.cpu().numpy(), 121 + b)
    if kind in ("bp2ht", "iht"):
        fresh = bht.HashTable(cfg, 0)
        host_keys = keys.keys.cpu().numpy()
        chunk = (DESK_N + 7) // 8
        where = {}
        for w in range(8):
            part = d_keys[w * chunk:(w + 1) * chunk]
            assert fresh.insert(part, bht.values_for_keys(part)).success
            store = fresh.download_store()
            slot_keys = (store & np.uint64(0xFFFFFFFF)).astype(np.uint32)
            occupied = np.flatnonzero(store != np.uint64(0xFFFFFFFFFFFFFFFF))
            order = np.argsort(slot_keys[occupied], kind="stable")
            sorted_keys, sorted_slots = slot_keys[occupied][order], occupied[order]
            mine = host_keys[w * chunk:(w + 1) * chunk]
            pos = np.searchsorted(sorted_keys, mine)
            assert np.array_equal(sorted_keys[pos], mine)
            where[w] = sorted_slots[pos]
            for earlier in range(w):   # stability: what was placed by an earlier batch is still exactly there
                old = host_keys[earlier * chunk:(earlier + 1) * chunk]
                assert np.array_equal(slot_keys[where[earlier]], old)
        fresh.close()


def test_criterion_10_sector_model_arithmetic(bht):
    """acceptance.cpp:459-469 (host arithmetic, exact)."""
    assert bht.predict_sectors("bcht", 16, 1.0, bht.OP_FIND) == 4.0
    assert bht.predict_sectors("bcht", 16, 3.0, bht.OP_FIND) == 12.0
    assert bht.predict_sectors("bcht", 16, 1.0, bht.OP_INSERT) == 5.0
