"""Host mirror of the reference's experiment protocol (proj/include/bht/experiments.hpp, proj/src/experiments.cpp) and
of its wire formats (config JSON core.cpp:70-109, result CSV / JSON experiments.cpp:232-268), driving the GPU tables.

Same names, same seed derivations, same record layout, so the outputs diff against the reference's `htbench`:
  * hash constants per build attempt: make_config(..., seed = mix_seed(cell.seed, 0x100 + attempt))   (experiments.cpp:70-72)
  * keys:    generate_keys(mix_seed(cell.seed, 0x6b657973), n)                                          (experiments.cpp:59)
  * queries: generate_queries(keys, ratio, n, mix_seed(cell.seed, 0x200 + r))                           (experiments.cpp:88-89)
  * cells:   cell_seed(base, i) = mix_seed(base, 0x63656c6c + i)                                        (experiments.cpp:27-29)
  * success-rate builds: make_config(..., seed = mix_seed(cell_seed(seed, cell), t))                    (experiments.cpp:123-124)
Probe means come from the device probe counters (one probe per bucket read = probe_stats.hpp:12-31); `sectors` is the
reference's analytic sector model (sector_model.hpp:26-31) applied to them.  What differs from the CPU reference is
what the north star allows to differ: a bulk build is concurrent, so which builds fail at the edge of a variant's
load range, and the third decimal of a probe mean, are those of a different (equally valid) insertion order.
"""
from __future__ import annotations

import json
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, TextIO

import numpy as np
import torch

from . import workload
from ._lib import Config
from .table import KIND_NAMES, OP_FIND, OP_INSERT, HashTable, make_config, mix_seed, predict_sectors, values_for_keys

KINDS = {name: code for code, name in KIND_NAMES.items()}  # parse_table_kind (core.cpp:20-26): the four printed names only
SCENARIOS = ("load_factor_sweep", "key_count_sweep", "positive_ratio_sweep", "success_rate", "probe_analysis")
HASH_PRIME = 4294967291
RESULT_CSV_HEADER = "kind,b,threshold_pct,n,realized_lf,op,positive_ratio,mean_probes,ops_per_sec,successes,failures,seed"


def parse_scenario(name: str) -> Optional[str]:
    return name if name in SCENARIOS else None


def cell_seed(base: int, cell_index: int) -> int:
    return mix_seed(base, 0x63656C6C + cell_index)


def format_double(v: float) -> str:
    """std::snprintf("%.6g") (experiments.cpp:21-25)."""
    return "%.6g" % v


# ---- config JSON (core.cpp:70-109) -------------------------------------------------------------------------------

def config_to_json(cfg: Config) -> str:
    """config_to_json: nlohmann dump(2) = keys in alphabetical order, two-space indent."""
    h = int(cfg.n_hashes)
    doc = {
        "kind": KIND_NAMES[int(cfg.kind)], "num_buckets": int(cfg.num_buckets), "bucket_size": int(cfg.bucket_size),
        "capacity": int(cfg.capacity),
        "hash_params": [{"alpha": int(cfg.alpha[i]), "beta": int(cfg.beta[i]), "prime": HASH_PRIME, "range": int(cfg.range[i])}
                        for i in range(h)],
        "threshold": int(cfg.threshold), "max_chain": int(cfg.max_chain), "seed": int(cfg.seed),
    }
    return json.dumps(doc, indent=2, sort_keys=True)


def config_from_json(text: str) -> Config:
    """config_from_json: ValueError where the reference throws invalid_argument."""
    from .table import hash_count
    j = json.loads(text)
    if j["kind"] not in KINDS:
        raise ValueError("config_from_json: unknown table kind")
    cfg = Config()
    cfg.kind = KINDS[j["kind"]]
    cfg.num_buckets = int(j["num_buckets"])
    cfg.bucket_size = int(j["bucket_size"])
    cfg.capacity = int(j["capacity"])
    params = j["hash_params"]
    for p in params:
        if int(p["prime"]) != HASH_PRIME:
            raise ValueError("config_from_json: unexpected prime")
    if len(params) != hash_count(cfg.kind):
        raise ValueError("config_from_json: wrong hash_params count for kind")
    cfg.n_hashes = len(params)
    for i, p in enumerate(params):
        cfg.alpha[i], cfg.beta[i], cfg.range[i] = int(p["alpha"]), int(p["beta"]), int(p["range"])
    cfg.threshold = int(j["threshold"])
    cfg.max_chain = int(j["max_chain"])
    cfg.seed = int(j["seed"])
    if cfg.capacity != cfg.num_buckets * cfg.bucket_size:
        raise ValueError("config_from_json: capacity mismatch")
    return cfg


# ---- spec / records (experiments.hpp) ----------------------------------------------------------------------------

@dataclass
class KindParams:
    kind: str = "bcht"
    bucket_size: int = 16
    threshold_pct: int = 80  # iht only

    def threshold_slots(self) -> Optional[int]:
        if self.kind != "iht":
            return None
        return self.bucket_size * self.threshold_pct // 100


@dataclass
class ExperimentSpec:
    scen: str = "probe_analysis"
    kinds: List[KindParams] = field(default_factory=list)
    n_grid: List[int] = field(default_factory=list)
    lf_grid: List[float] = field(default_factory=list)
    positive_ratios: List[float] = field(default_factory=list)
    trials: int = 10
    max_failures: int = 50
    success_trials: int = 200
    seed: int = 0
    mode: str = "seq"              # build_options: kept for file compatibility; a GPU build is always bulk
    workers: int = 0
    iht_prose_fallback: bool = False
    max_chain: Optional[int] = None


def spec_to_json(spec: ExperimentSpec) -> str:
    doc = {
        "scenario": spec.scen,
        "kinds": [{"kind": k.kind, "bucket_size": k.bucket_size, "threshold_pct": k.threshold_pct} for k in spec.kinds],
        "n_grid": list(spec.n_grid), "lf_grid": list(spec.lf_grid), "positive_ratios": list(spec.positive_ratios),
        "trials": spec.trials, "max_failures": spec.max_failures, "success_trials": spec.success_trials, "seed": spec.seed,
        "mode": spec.mode, "workers": spec.workers, "iht_prose_fallback": spec.iht_prose_fallback, "max_chain": spec.max_chain,
    }
    return json.dumps(doc, indent=2, sort_keys=True)


def spec_from_json(text: str) -> ExperimentSpec:
    j = json.loads(text)
    if parse_scenario(j["scenario"]) is None:
        raise ValueError("spec_from_json: unknown scenario")
    spec = ExperimentSpec(scen=j["scenario"])
    for k in j["kinds"]:
        if k["kind"] not in KINDS:
            raise ValueError("spec_from_json: unknown table kind")
        spec.kinds.append(KindParams(k["kind"], int(k["bucket_size"]), int(k.get("threshold_pct", 80))))
    spec.n_grid = [int(x) for x in j["n_grid"]]
    spec.lf_grid = [float(x) for x in j["lf_grid"]]
    spec.positive_ratios = [float(x) for x in j.get("positive_ratios", [])]
    for name in ("trials", "max_failures", "success_trials", "seed", "workers"):
        if name in j:
            setattr(spec, name, int(j[name]))
    if "mode" in j:
        spec.mode = "par" if j["mode"] == "par" else "seq"
    if "iht_prose_fallback" in j:
        spec.iht_prose_fallback = bool(j["iht_prose_fallback"])
    if j.get("max_chain") is not None:
        spec.max_chain = int(j["max_chain"])
    return spec


@dataclass
class ResultRecord:
    kind: str = "bcht"
    b: int = 0
    threshold_pct: Optional[int] = None
    n: int = 0
    realized_lf: float = 0.0
    op: str = ""                      # "insert", "find" or "build"
    positive_ratio: Optional[float] = None
    mean_probes: float = 0.0
    ops_per_sec: float = 0.0
    successes: int = 0
    failures: int = 0
    seed: int = 0
    budget_exhausted: bool = False

    def sectors(self) -> float:
        """predict_sectors (sector_model.hpp:26-31) for this record's probe mean; 0 for "build" rows."""
        if self.op == "build":
            return 0.0
        return predict_sectors(self.kind, self.b, self.mean_probes, OP_INSERT if self.op == "insert" else OP_FIND)


@dataclass
class ExperimentResult:
    records: List[ResultRecord] = field(default_factory=list)
    wall_seconds: float = 0.0

    def any_budget_exhausted(self) -> bool:
        return any(r.budget_exhausted for r in self.records)


def write_csv(out: TextIO, result: ExperimentResult) -> None:
    """write_csv (experiments.cpp:232-243): same header, same column formats."""
    out.write(RESULT_CSV_HEADER + "\n")
    for r in result.records:
        out.write(",".join([
            r.kind, str(r.b), "" if r.threshold_pct is None else str(r.threshold_pct), str(r.n), format_double(r.realized_lf), r.op,
            "" if r.positive_ratio is None else format_double(r.positive_ratio), format_double(r.mean_probes),
            format_double(r.ops_per_sec), str(r.successes), str(r.failures), str(r.seed)]) + "\n")


def write_json(out: TextIO, result: ExperimentResult) -> None:
    """write_json (experiments.cpp:245-268)."""
    recs = [{"kind": r.kind, "b": r.b, "threshold_pct": r.threshold_pct, "n": r.n, "realized_lf": r.realized_lf, "op": r.op,
             "positive_ratio": r.positive_ratio, "mean_probes": r.mean_probes, "ops_per_sec": r.ops_per_sec,
             "successes": r.successes, "failures": r.failures, "seed": r.seed, "budget_exhausted": r.budget_exhausted}
            for r in result.records]
    out.write(json.dumps({"records": recs, "wall_seconds": result.wall_seconds}, indent=2, sort_keys=True) + "\n")


# ---- the trials / failure-budget protocol (experiments.cpp:51-112) ------------------------------------------------

@dataclass
class TrialCell:
    params: KindParams = field(default_factory=KindParams)
    n: int = 0
    lf: float = 0.0
    positive_ratios: Sequence[float] = ()
    trials: int = 10
    max_failures: int = 50
    seed: int = 0
    max_chain: Optional[int] = None
    iht_prose_fallback: bool = False
    preloaded_keys: Optional[workload.KeySet] = None  # reused across cells when its size matches


@dataclass
class TrialOutcome:
    successes: int = 0
    failures: int = 0
    budget_exhausted: bool = False
    realized_lf: float = 0.0
    insert_mean_probes: float = 0.0
    insert_ops_per_sec: float = 0.0
    find_mean_probes: List[float] = field(default_factory=list)
    find_ops_per_sec: List[float] = field(default_factory=list)


def _device_keys(keys: workload.KeySet, device: int) -> torch.Tensor:
    k = keys.keys
    if isinstance(k, torch.Tensor):
        return k.to(f"cuda:{device}").view(torch.int32)
    return torch.from_numpy(np.ascontiguousarray(k).view(np.int32)).to(f"cuda:{device}")


def _timed(fn, device: int) -> float:
    """Device seconds of fn() on the current stream (CUDA events; the reference uses steady_clock around the call)."""
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(torch.cuda.current_stream(device))
    fn()
    b.record(torch.cuda.current_stream(device))
    b.synchronize()
    return a.elapsed_time(b) * 1e-3


def run_trial(cell: TrialCell, device: int = 0) -> TrialOutcome:
    """run_trial: fresh hash constants per attempt, build until `trials` successes or the failure budget runs out; on
    each success one bulk find of q = n queries per requested ratio."""
    out = TrialOutcome()
    ratios = list(cell.positive_ratios)
    out.find_mean_probes = [0.0] * len(ratios)
    out.find_ops_per_sec = [0.0] * len(ratios)
    keys = cell.preloaded_keys
    if keys is None or keys.size() != cell.n:
        keys = workload.generate_keys(mix_seed(cell.seed, 0x6B657973), cell.n, device=device)
    d_keys = _device_keys(keys, device)
    d_vals = None  # keys-only build: the library pairs every key with value_for_key (table.cpp:234) on the device

    ins_probes = ins_ops = 0
    ins_seconds = 0.0
    find_probes = [0] * len(ratios)
    find_ops = [0] * len(ratios)
    find_seconds = [0.0] * len(ratios)
    queries: List[Optional[torch.Tensor]] = [None] * len(ratios)
    out_buf = torch.empty(cell.n, dtype=torch.int32, device=f"cuda:{device}") if ratios else None

    attempt = 0
    while out.successes < cell.trials and out.failures < cell.max_failures:
        cfg = make_config(cell.params.kind, cell.n, cell.lf, cell.params.bucket_size, cell.params.threshold_slots(),
                          mix_seed(cell.seed, 0x100 + attempt), cell.max_chain)
        attempt += 1
        out.realized_lf = cell.n / cfg.capacity
        table = HashTable(cfg, device)
        try:
            if cell.iht_prose_fallback and cell.params.kind == "iht":
                table.set_iht_prose_fallback(True)
            elapsed = _timed(lambda: table.insert(d_keys, d_vals, want_result=False), device)
            built = table.last_insert_result()
            if not built.success:
                out.failures += 1
                continue
            out.successes += 1
            ins_probes += built.probes
            ins_ops += built.attempted
            ins_seconds += elapsed
            for r, ratio in enumerate(ratios):
                if queries[r] is None:  # the query set depends on (keys, ratio, seed) only: one generation per cell
                    qs = workload.generate_queries(keys, ratio, cell.n, mix_seed(cell.seed, 0x200 + r), device=device)
                    queries[r] = torch.from_numpy(qs.keys.view(np.int32)).to(f"cuda:{device}")
                stats_box = []
                find_seconds[r] += _timed(lambda: stats_box.append(table.find(queries[r], out_buf, want_stats=True)[1]), device)
                find_probes[r] += stats_box[0].probes
                find_ops[r] += cell.n
        finally:
            table.close()

    out.budget_exhausted = out.successes < cell.trials
    out.insert_mean_probes = ins_probes / ins_ops if ins_ops else 0.0
    if ins_seconds > 0.0:
        out.insert_ops_per_sec = ins_ops / ins_seconds
    for r in range(len(ratios)):
        out.find_mean_probes[r] = find_probes[r] / find_ops[r] if find_ops[r] else 0.0
        if find_seconds[r] > 0.0:
            out.find_ops_per_sec[r] = find_ops[r] / find_seconds[r]
    return out


@dataclass
class SuccessRatePoint:
    lf: float = 0.0
    realized_lf: float = 0.0
    successes: int = 0
    trials: int = 0

    def fraction(self) -> float:
        return 0.0 if self.trials == 0 else self.successes / self.trials


@dataclass
class SuccessRateResult:
    points: List[SuccessRatePoint] = field(default_factory=list)
    max_load_factor: Optional[float] = None  # highest grid load factor with >= 99 % successes


def run_success_rate(params: KindParams, n: int, lf_grid: Sequence[float], success_trials: int, seed: int,
                     max_chain: Optional[int] = None, device: int = 0, iht_prose_fallback: bool = False) -> SuccessRateResult:
    """run_success_rate (experiments.cpp:114-146): `success_trials` builds per load factor, fresh constants each."""
    result = SuccessRateResult()
    keys = workload.generate_keys(mix_seed(seed, 0x6B657973), n, device=device)
    d_keys = _device_keys(keys, device)
    d_vals = None  # keys-only build (table.cpp:234)
    for cell, lf in enumerate(lf_grid):
        point = SuccessRatePoint(lf=lf, trials=success_trials)
        table = None
        for t in range(success_trials):
            cfg = make_config(params.kind, n, lf, params.bucket_size, params.threshold_slots(), mix_seed(cell_seed(seed, cell), t),
                              max_chain)
            point.realized_lf = n / cfg.capacity
            table = HashTable(cfg, device)
            try:
                if iht_prose_fallback and params.kind == "iht":
                    table.set_iht_prose_fallback(True)
                point.successes += bool(table.insert(d_keys, d_vals).success)
            finally:
                table.close()
        result.points.append(point)
    for p in result.points:
        if p.fraction() >= 0.99 and (result.max_load_factor is None or p.lf > result.max_load_factor):
            result.max_load_factor = p.lf
    return result


def run_experiment(spec: ExperimentSpec, device: int = 0) -> ExperimentResult:
    """run_experiment (experiments.cpp:153-230): one record per (cell, op, positive ratio)."""
    if not spec.kinds:
        raise ValueError("run_experiment: no table kinds requested")
    if not spec.n_grid:
        raise ValueError("run_experiment: empty key-count grid")
    if not spec.lf_grid:
        raise ValueError("run_experiment: empty load-factor grid")
    if spec.trials < 1:
        raise ValueError("run_experiment: trials must be at least 1")
    result = ExperimentResult()
    start = time.perf_counter()
    cell_index = 0
    for params in spec.kinds:
        tpct = params.threshold_pct if params.kind == "iht" else None
        for n in spec.n_grid:
            if spec.scen == "success_rate":
                sr = run_success_rate(params, n, spec.lf_grid, spec.success_trials, mix_seed(spec.seed, cell_index),
                                      spec.max_chain, device, spec.iht_prose_fallback)
                cell_index += 1
                for p in sr.points:
                    result.records.append(ResultRecord(params.kind, params.bucket_size, tpct, n, p.realized_lf, "build", None, 0.0, 0.0,
                                                       p.successes, p.trials - p.successes, spec.seed))
                continue
            for lf in spec.lf_grid:
                cell = TrialCell(params, n, lf, list(spec.positive_ratios), spec.trials, spec.max_failures,
                                 cell_seed(spec.seed, cell_index), spec.max_chain, spec.iht_prose_fallback)
                cell_index += 1
                o = run_trial(cell, device)
                ins = ResultRecord(params.kind, params.bucket_size, tpct, n, o.realized_lf, "insert", None, o.insert_mean_probes,
                                   o.insert_ops_per_sec, o.successes, o.failures, spec.seed, o.budget_exhausted)
                result.records.append(ins)
                for r, ratio in enumerate(spec.positive_ratios):
                    result.records.append(ResultRecord(params.kind, params.bucket_size, tpct, n, o.realized_lf, "find", ratio,
                                                       o.find_mean_probes[r], o.find_ops_per_sec[r], o.successes, o.failures,
                                                       spec.seed, o.budget_exhausted))
    result.wall_seconds = time.perf_counter() - start
    return result
