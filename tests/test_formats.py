"""CPU-side checks of the wire / on-disk formats and the experiment records of the host layer against
the reference's own writers (proj/src/core.cpp:70-109, proj/src/experiments.cpp:232-312, proj/src/keygen.cpp:100-125),
reached through oracle/_ref.  No GPU call is made: configs, JSON, CSV and key files are host-only."""
import io
import json
import os

import numpy as np
import pytest

from oracle import binding


@pytest.fixture(scope="module")
def ex():
    from paper_2108_07232_b200 import experiments
    return experiments


@pytest.fixture(scope="module")
def refx(ref):
    if not ref.has_experiments():
        pytest.skip("oracle/_ref was compiled without experiments.cpp (no nlohmann/json.hpp)")
    return ref


CONFIG_CASES = [("bcht", 50_000_000, 0.9, 16, None, 257), ("1cht", 1000, 0.8, 1, None, 3), ("bp2ht", 12345, 0.6, 32, None, 0),
                ("iht", 99_999, 0.86, 16, 6, 2**63 + 11), ("iht", 1000, 0.8, 64, None, 5)]


@pytest.mark.parametrize("kind,n,lf,b,t,seed", CONFIG_CASES)
def test_config_json_is_the_reference_text(bht, ex, refx, kind, n, lf, b, t, seed):
    cfg = bht.make_config(kind, n, lf, b, threshold=t, seed=seed)
    rcfg = refx.make_config(binding.KINDS[kind], n, lf, b, threshold=t, seed=seed)
    text = ex.config_to_json(cfg)
    assert text == refx.config_to_json(rcfg)           # byte for byte (nlohmann dump(2): sorted keys, 2-space indent)
    back = ex.config_from_json(text)
    assert bytes(back) == bytes(cfg)
    assert bytes(refx.config_from_json(text)) == bytes(rcfg) == bytes(cfg)


def test_config_json_rejections(bht, ex):
    """config_from_json throws invalid_argument (core.cpp:83-107): unknown kind, wrong prime, wrong hash count,
    capacity mismatch."""
    good = json.loads(ex.config_to_json(bht.make_config("bcht", 1000, 0.9, 16, seed=1)))
    for mutate in (lambda j: j.update(kind="cuckoo"), lambda j: j["hash_params"][0].update(prime=4294967295),
                   lambda j: j["hash_params"].pop(), lambda j: j.update(capacity=j["capacity"] + 1)):
        j = json.loads(json.dumps(good))
        mutate(j)
        with pytest.raises(ValueError):
            ex.config_from_json(json.dumps(j))


def test_spec_json_round_trip_and_reference_canonical_form(ex, refx):
    """The spec of proj/tests/test_experiments.cpp:200-226, through both implementations."""
    spec = ex.ExperimentSpec(scen="success_rate", kinds=[ex.KindParams("iht", 32, 60), ex.KindParams("1cht", 1, 80)],
                             n_grid=[1000, 2000], lf_grid=[0.5, 0.9], positive_ratios=[1.0, 0.5], trials=4, max_failures=9,
                             success_trials=33, seed=123456789, mode="par", workers=3, iht_prose_fallback=True, max_chain=77)
    text = ex.spec_to_json(spec)
    assert ex.spec_from_json(text) == spec
    assert json.loads(refx.spec_roundtrip(text)) == json.loads(text)   # the reference parses and re-emits the same document
    # defaults for the optional members (experiments.cpp:286-306)
    minimal = ex.spec_from_json('{"scenario": "probe_analysis", "kinds": [{"kind": "bcht", "bucket_size": 16}], "n_grid": [10], "lf_grid": [0.5]}')
    ref_min = json.loads(refx.spec_roundtrip('{"scenario": "probe_analysis", "kinds": [{"kind": "bcht", "bucket_size": 16}], "n_grid": [10], "lf_grid": [0.5]}'))
    assert json.loads(ex.spec_to_json(minimal)) == ref_min
    with pytest.raises(ValueError):
        ex.spec_from_json('{"scenario": "nope", "kinds": [], "n_grid": [], "lf_grid": []}')
    with pytest.raises(ValueError):
        ex.spec_from_json('{"scenario": "probe_analysis", "kinds": [{"kind": "x", "bucket_size": 1}], "n_grid": [1], "lf_grid": [0.5]}')


def parse_reference_csv(ex, text):
    lines = text.strip("\n").split("\n")
    assert lines[0] == ex.RESULT_CSV_HEADER
    recs = []
    for line in lines[1:]:
        kind, b, tp, n, lf, op, ratio, probes, ops, succ, fail, seed = line.split(",")
        recs.append(ex.ResultRecord(kind, int(b), int(tp) if tp else None, int(n), float(lf), op, float(ratio) if ratio else None,
                                    float(probes), float(ops), int(succ), int(fail), int(seed)))
    return recs


def test_csv_writer_reproduces_the_reference_file(ex, refx):
    """A CSV written by the reference's write_csv (a real CPU run of run_experiment on a tiny grid), parsed into
    ResultRecords and written again by the product's writer, is the same text: header, column order, '%.6g' numbers,
    empty threshold_pct / positive_ratio cells (experiments.hpp:81-82, experiments.cpp:232-243)."""
    spec = ex.ExperimentSpec(scen="probe_analysis", kinds=[ex.KindParams("bcht", 16, 80), ex.KindParams("iht", 16, 75)],
                             n_grid=[3000], lf_grid=[0.5, 0.8], positive_ratios=[1.0, 0.0], trials=2, max_failures=5, seed=42)
    text = refx.run_experiment(ex.spec_to_json(spec), "csv")
    recs = parse_reference_csv(ex, text)
    assert len(recs) == 2 * 2 * 3   # kinds x lf cells x (insert + 2 find ratios)   (test_experiments.cpp:63-83)
    for r in recs:
        r.ops_per_sec = 0.0  # timing column: informational only (experiments.hpp:66-67)
    out = io.StringIO()
    ex.write_csv(out, ex.ExperimentResult(recs))
    want = "\n".join(",".join(c if i != 8 else "0" for i, c in enumerate(line.split(","))) if n else line
                     for n, line in enumerate(text.strip("\n").split("\n"))) + "\n"
    assert out.getvalue() == want
    # success-rate runs produce "build" rows with zero probe means
    sr = ex.ExperimentSpec(scen="success_rate", kinds=[ex.KindParams("bcht", 16, 80)], n_grid=[2000], lf_grid=[0.1, 0.5],
                           success_trials=3, seed=7)
    sr_recs = parse_reference_csv(ex, refx.run_experiment(ex.spec_to_json(sr), "csv"))
    assert [r.op for r in sr_recs] == ["build", "build"] and all(r.successes == 3 and r.failures == 0 for r in sr_recs)
    # JSON writer: same members as the reference's records (experiments.cpp:245-268)
    doc = json.loads(refx.run_experiment(ex.spec_to_json(sr), "json"))
    mine = io.StringIO()
    ex.write_json(mine, ex.ExperimentResult(sr_recs, 0.0))
    mine_doc = json.loads(mine.getvalue())
    assert set(mine_doc) == set(doc) == {"records", "wall_seconds"}
    assert [set(r) for r in mine_doc["records"]] == [set(r) for r in doc["records"]]
    for a, b in zip(mine_doc["records"], doc["records"]):
        assert {k: v for k, v in a.items() if k != "ops_per_sec"} == {k: v for k, v in b.items() if k != "ops_per_sec"}


def test_sector_report_matches_the_reference_model(bht, ex, ref):
    """ResultRecord.sectors() = predict_sectors (sector_model.hpp:26-31) for insert / find rows, every kind."""
    for kind, b, probes in (("bcht", 16, 1.1085), ("bcht", 8, 1.2), ("1cht", 1, 2.7538), ("bp2ht", 32, 2.0), ("iht", 16, 1.48)):
        for op in ("insert", "find"):
            rec = ex.ResultRecord(kind, b, None, 1000, 0.9, op, None, probes)
            assert rec.sectors() == ref.predict_sectors(kind, b, probes, op)
    assert ex.ResultRecord(op="build").sectors() == 0.0


def test_key_file_round_trip_and_byte_order(bht, ref, tmp_path):
    """save_keys / load_keys (keygen.cpp:100-125): flat little-endian u32; a trailing partial word is ignored."""
    from paper_2108_07232_b200 import workload
    keys = ref.generate_keys(23, 1000)
    path = tmp_path / "keys.bin"
    workload.save_keys(str(path), keys)
    raw = path.read_bytes()
    assert raw == keys.astype("<u4").tobytes()
    loaded = workload.load_keys(str(path), seed=23)
    assert loaded.seed == 23 and np.array_equal(loaded.keys, keys)
    path.write_bytes(raw + b"\x01\x02")
    assert np.array_equal(workload.load_keys(str(path)).keys, keys)
    workload.save_keys(str(path), np.empty(0, dtype=np.uint32))
    assert workload.load_keys(str(path)).keys.size == 0
    with pytest.raises(OSError):
        workload.load_keys(str(tmp_path / "missing.bin"))
    with pytest.raises(OSError):
        workload.save_keys(str(tmp_path / "no_such_dir" / "k.bin"), keys)


# ---- committed fixtures (tests/golden/reference_formats.json, made by tests/golden/make_golden_workload.py) ----------

GOLDEN_FORMATS = os.path.join(os.path.dirname(__file__), "golden", "reference_formats.json")


def test_golden_config_json_and_csv(bht, ex):
    """The same pins without oracle/_ref: config JSON text per (kind, n, lf, b, t, seed), and the reference's CSV of one
    tiny run reproduced by write_csv from its own parsed records (ops_per_sec column aside)."""
    doc = json.load(open(GOLDEN_FORMATS))
    for case in doc["configs"]:
        kind, n, lf, b, t, seed = case["args"]
        assert ex.config_to_json(bht.make_config(kind, n, lf, b, threshold=t, seed=seed)) == case["json"]
        assert ex.config_to_json(ex.config_from_json(case["json"])) == case["json"]
    recs = parse_reference_csv(ex, doc["csv"])
    assert [r.op for r in recs[:3]] == ["insert", "find", "find"] and recs[0].positive_ratio is None
    assert all(r.threshold_pct == (75 if r.kind == "iht" else None) for r in recs)
    out = io.StringIO()
    ex.write_csv(out, ex.ExperimentResult(recs))
    assert out.getvalue() == doc["csv"]          # ops_per_sec too: '%.6g' of the parsed double is the same text
    spec = ex.spec_from_json(json.dumps(doc["spec"]))
    assert (spec.trials, spec.max_failures, spec.seed, [k.threshold_pct for k in spec.kinds]) == (2, 5, 42, [80, 75])
    mine = io.StringIO()
    ex.write_json(mine, ex.ExperimentResult(recs[:1]))
    assert sorted(json.loads(mine.getvalue())["records"][0]) == doc["result_json_members"]
