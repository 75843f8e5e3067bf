#!/usr/bin/env python
"""bench.py — BASELINE.json's metric on B200: bulk insert & bulk find MKeys/s.

A step is one pass of the hot path over one batch: bulk BUILD (clear the store + insert n pairs) followed by
bulk FIND of n queries (100 % positive), on the configuration the metric is quoted on: BCHT b=16, 50 M
unique uniformly distributed 32-bit keys (MT19937), load factor 0.9.  `value` = 2n keys / step time with the
inputs resident in HBM; `e2e` = the same pass through the C ABI with HOST (pinned) buffers, PCIe copies inside
the timed region — as the reference's harness calls it: build(keys, cfg), values = value_for_key(key), so only keys
and queries cross PCIe (`e2e.explicit_values`: the same with caller-supplied values).  The other positive fractions (50 %, 0 %) and the per-kernel times are reported in `detail`.

    python bench.py [--gpus N] [--steps K] [--warmup W]            the CUDA path
    python bench.py --impl reference ...                            the reference CPU implementation (oracle/_ref)

N > 1 (torchrun, one rank per GPU): the sharded table — 50 M keys per GPU generated on the device, NCCL
all-to-all routing inside the timed region, weak scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KIND, B, LF, N_KEYS, SEED, THRESHOLD = "bcht", 16, 0.9, 50_000_000, 1, None
METRIC = "insert & find MKeys/s, BCHT b=16, 50M keys, LF 0.9"
HEADLINE = True

# BASELINE.json's configurations, by name (--config); `kind:b:lf[:t]` names any other cell.  The default is the one the
# metric is quoted on (configs[1]'s family at LF 0.9, see METRIC).
CONFIGS = {
    "headline": ("bcht", 16, 0.9, None),
    "bcht08": ("bcht", 16, 0.8, None), "bcht09": ("bcht", 16, 0.9, None), "bcht099": ("bcht", 16, 0.99, None),
    "1cht08": ("1cht", 1, 0.8, None), "1cht09": ("1cht", 1, 0.9, None),
    "bp2ht06": ("bp2ht", 16, 0.6, None), "bp2ht07": ("bp2ht", 16, 0.7, None), "bp2ht08": ("bp2ht", 16, 0.8, None),
    "bp2ht084": ("bp2ht", 16, 0.84, None), "bp2ht09": ("bp2ht", 16, 0.9, None), "bp2ht099": ("bp2ht", 16, 0.99, None),
    "iht08": ("iht", 16, 0.8, 12), "iht09": ("iht", 16, 0.9, 12), "iht099": ("iht", 16, 0.99, 12),
}


def select_config(name: str):
    global KIND, B, LF, THRESHOLD, METRIC, HEADLINE
    if name in CONFIGS:
        KIND, B, LF, THRESHOLD = CONFIGS[name]
    else:
        parts = name.split(":")
        KIND, B, LF = parts[0], int(parts[1]), float(parts[2])
        THRESHOLD = int(parts[3]) if len(parts) > 3 else (int(0.8 * B) if KIND == "iht" else None)
    HEADLINE = (KIND, B, LF) == ("bcht", 16, 0.9)
    t = f", t={THRESHOLD}" if KIND == "iht" else ""
    METRIC = f"insert & find MKeys/s, {KIND.upper()} b={B}{t}, 50M keys, LF {LF}"  # the headline: BASELINE.json's metric string


def csrc_stamp() -> str:
    """Hash of the kernel sources: profiles/traffic.json is only quoted for the sources it was captured from."""
    import glob
    import hashlib
    h = hashlib.sha1()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2108_07232_b200", "csrc", "*.cu*")) +
                    glob.glob(os.path.join(ROOT, "paper_2108_07232_b200", "csrc", "*.h"))):
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


KEYS_STREAM, QUERY_STREAM = 0x6B657973, 0x200  # the reference harness's seed streams (experiments.cpp:59,88-89)


def make_values(n: int, seed: int):
    """n sentinel-free u32 values from a second MT19937 stream."""
    rng = np.random.Generator(np.random.MT19937(seed ^ 0x76616C73))
    v = rng.integers(0, 0xFFFFFFFF, size=n, dtype=np.uint32)  # high is exclusive: never the sentinel
    return v


def make_workload(n: int, seed: int):
    """(--workload numpy) n present + n absent unique sentinel-free u32 keys and n values from MT19937 streams."""
    rng = np.random.Generator(np.random.MT19937(seed))
    raw = rng.integers(0, 0xFFFFFFFF, size=int(2 * n * 1.02) + 1024, dtype=np.uint32)
    raw.sort()
    keep = np.empty(raw.size, dtype=bool)
    keep[0] = True
    np.not_equal(raw[1:], raw[:-1], out=keep[1:])
    uniq = raw[keep]
    assert uniq.size >= 2 * n
    rng.shuffle(uniq)
    values = rng.integers(0, 0xFFFFFFFF, size=n, dtype=np.uint32)
    return uniq[:n].copy(), uniq[n:2 * n].copy(), values


class StdoutToStderr:
    """Everything written to fd 1 inside the block goes to stderr: NCCL announces its version on stdout when the first
    communicator comes up, and stdout carries exactly one JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region, every ~2 ms from a host thread
    through NVML (the timed region of the default run lasts tens of milliseconds, too short for `nvidia-smi -lms`);
    falls back to one `nvidia-smi` query per sample when NVML cannot be loaded."""

    Q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"

    def __init__(self, gpu_index: int, uuid: str | None = None):
        self.gpu, self.uuid = gpu_index, uuid
        self.samples, self.reason_bits = [], 0
        self.sm_max = None
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None
        self._handle = None
        try:
            import pynvml
            pynvml.nvmlInit()
            try:
                self._handle = pynvml.nvmlDeviceGetHandleByUUID(uuid) if uuid else pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            except pynvml.NVMLError:
                self._handle = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.sm_max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._handle, pynvml.NVML_CLOCK_SM))
            self._nvml = pynvml
        except Exception:  # noqa: BLE001  (no NVML on this host: nvidia-smi below)
            self._nvml = None

    def _sample_once(self):
        if self._nvml is not None:
            nv = self._nvml
            self.samples.append(float(nv.nvmlDeviceGetClockInfo(self._handle, nv.NVML_CLOCK_SM)))
            self.reason_bits |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._handle))
            return
        r = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True, timeout=10)
        p = [x.strip() for x in r.stdout.strip().split(",")]
        self.samples.append(float(p[0]))
        self.sm_max = float(p[1])
        self.reason_bits |= int(p[2], 16)

    def _loop(self):
        while not self._stop.is_set():
            try:
                self._sample_once()
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.002)

    def start(self):
        self._thread = threading.Thread(target=self._loop, daemon=True)
        self._thread.start()

    def sample_until(self, event):
        """Samples from the calling thread while the GPU works towards `event` (a recorded torch.cuda.Event): the steps
        of the timed region are enqueued asynchronously, so the host is free exactly while the device is under load."""
        while not event.query():
            try:
                self._sample_once()
            except Exception:  # noqa: BLE001
                break

    def stop(self):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=15)
        # NVML clock-event reason bits (nvml.h): the ones that invalidate a run, plus the power cap (kept and noted)
        bits = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
                0x80: "hw_power_brake_slowdown"}
        reasons = sorted(name for bit, name in bits.items() if self.reason_bits & bit)
        sm = sorted(self.samples)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.sm_max, "reasons": reasons,
                "samples": len(sm), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ---- the reference arm: the reference's own CPU implementation -------------------------------------------------

def cpu_reference_pass(ref, cfg, present, queries, n_sample, threads):
    """One bounded pass of the reference CPU path: build() in parallel mode on all host threads
    (table.cpp:239-271) + the caller-side find_key loop chunked over the same threads."""
    table, out = ref.build(present[:n_sample], cfg, parallel=True, workers=threads)
    t_build = out["seconds"]
    _, hits, probes, t_find = table.find_bulk_timed(queries[:n_sample], threads)
    table.close()
    return t_build, t_find, out, hits


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import binding
    ref = binding.ref()
    threads = ref.hardware_concurrency()
    n = args.keys
    if args.workload == "reference":
        present = ref.generate_keys(ref.mix_seed(SEED, KEYS_STREAM), n)  # the harness's own key set (experiments.cpp:59)
    else:
        present, _absent, _values = make_workload(n, SEED)
    ocfg = make_ref_config(ref, n)
    # size the per-step sample so that the whole run ends within a few minutes
    t0 = time.time()
    probe_n = min(n, 2_000_000)
    tb, tf, _, _ = cpu_reference_pass(ref, ocfg, present, present, probe_n, threads)
    rate = 2 * probe_n / max(tb + tf, 1e-9)
    budget = 150.0
    n_sample = int(min(n, max(1_000_000, rate * budget / (args.steps + args.warmup) / 2)))
    for _ in range(args.warmup):
        cpu_reference_pass(ref, ocfg, present, present, n_sample, threads)
    times, tbs, tfs = [], [], []
    for _ in range(args.steps):
        tb, tf, out, hits = cpu_reference_pass(ref, ocfg, present, present, n_sample, threads)
        assert out["success"] and hits == n_sample
        times.append(tb + tf)
        tbs.append(tb)
        tfs.append(tf)
    total = sum(times)
    value = 2 * n_sample * args.steps / total / 1e6
    sample = (f"first {n_sample} of the {n} keys built into the full-size ({ocfg.capacity * 8 / 1e6:.0f} MB) table "
              f"with the reference's build(parallel, {threads} workers), then {n_sample} positive find_key calls "
              f"chunked over {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MKeys/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64 integer",
        "data": data_label(args),
        "config": workload_config(n, args.gpus, ocfg.capacity * 8 / 1e6),
        "cpu_baseline": {"value": value, "unit": "MKeys/s", "cores": threads, "kind": "reference", "sample": sample,
                         "insert_mkeys": n_sample * args.steps / sum(tbs) / 1e6,
                         "find_mkeys": n_sample * args.steps / sum(tfs) / 1e6},
        "e2e": {"value": value, "unit": "MKeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(line), flush=True)
    return 0


def make_ref_config(ref, n, attempt=0):
    from oracle import binding
    kw = {"threshold": THRESHOLD} if KIND == "iht" and THRESHOLD is not None else {}
    cfg = ref.make_config(binding.KINDS[KIND], n, LF, B, seed=ref.mix_seed(SEED, 0x100 + attempt), **kw)
    return cfg


def data_label(args):
    if args.workload == "reference":
        return ("synthetic: the reference harness's workload for seed 1 - generate_keys (unique uniform u32, mt19937_64) and "
                "generate_queries per positive ratio; values from a second MT19937 stream")
    return "synthetic: unique uniform u32 keys, MT19937"


def workload_config(n, gpus, table_mb=None):
    return {"workload": f"{KIND} b={B}, {n} unique u32 keys/values per GPU, load factor {LF}: bulk build then "
                        f"{n} positive bulk finds", "kind": KIND, "bucket_size": B, "load_factor": LF,
            "keys_per_gpu": n, "table_mb": table_mb, "l2": "table and inputs each exceed the 126 MB L2; no flush needed",
            "parallelism": "single table" if gpus == 1 else f"key-range sharded x{gpus}, NCCL all-to-all"}


# ---- the CUDA arm ------------------------------------------------------------------------------------------------

def run_cuda(args):
    import torch
    import torch.distributed as dist

    import paper_2108_07232_b200 as bht

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the CUDA arm has no CPU fallback (use --impl reference)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        with StdoutToStderr():
            dist.init_process_group("nccl", device_id=device)
    n = args.keys
    kw = {"threshold": THRESHOLD} if KIND == "iht" and THRESHOLD is not None else {}
    cfg_for = lambda attempt: bht.make_config(KIND, n, LF, B, seed=bht.mix_seed(SEED, 0x100 + attempt), **kw)  # noqa: E731
    cfg = cfg_for(0)  # hash constants per attempt as the reference's run_trial draws them (experiments.cpp:66-70)
    wl = workload_config(n, world)
    wl["table_mb"] = cfg.capacity * 8 / 1e6

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    stream = torch.cuda.current_stream()
    try:
        uuid = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    except Exception:  # noqa: BLE001
        uuid = None
    sampler = ClockSampler(local, uuid)

    if world == 1 and not args.sharded:
        if args.device_keys:
            # sizes where the MT19937 host generator is impractical (the 5*10^8-key shard of the 4-billion-key
            # configuration): keys / values from the device bijection, negatives = the next n counters
            dk, dv = bht.generate_unique_keys(SEED, 0, n, device=local)
            da = bht.generate_unique_keys(SEED, n, n, device=local, with_values=False)
            d_keys, d_vals, d_abs = dk.view(torch.int32), dv.view(torch.int32), da.view(torch.int32)
            present, values, absent = None, None, None
        elif args.workload == "reference":
            # exactly what the reference's run_trial would build and query for seed S = 1 (experiments.cpp:59,88-89),
            # generated through this library (element for element the reference's outputs, tests/test_gpu_workload.py)
            ks = bht.workload.generate_keys(bht.mix_seed(SEED, KEYS_STREAM), n, device=local)
            d_keys = ks.keys.view(torch.int32)
            present = d_keys.cpu().numpy().view(np.uint32)
            values = make_values(n, SEED)
            d_vals = torch.from_numpy(values.view(np.int32)).to(device)
            qsets = []
            for r, ratio in enumerate((1.0, 0.5, 0.0)):
                q = bht.workload.generate_queries(ks, ratio, n, bht.mix_seed(SEED, QUERY_STREAM + r), device=local)
                assert int(q.expected_present.sum()) == int(round(ratio * n))
                qsets.append(torch.from_numpy(q.keys.view(np.int32)).to(device))
            d_pos, d_mixed, d_abs = qsets
            absent = None
        else:
            present, absent, values = make_workload(n, SEED)
            d_keys = torch.from_numpy(present.view(np.int32)).to(device)
            d_vals = torch.from_numpy(values.view(np.int32)).to(device)
            d_abs = torch.from_numpy(absent.view(np.int32)).to(device)
        d_out = torch.empty(n, dtype=torch.int32, device=device)
        half = n // 2
        if args.device_keys or args.workload != "reference":
            d_pos = d_keys
            d_mixed = torch.cat([d_keys[:half], d_abs[:n - half]])[torch.randperm(n, device=device)].contiguous()
        # the reference's trial protocol retries a failed build with fresh hash constants (experiments.cpp:62-84);
        # the first attempt that builds is the table that is timed (a cell that never builds is timed as it is)
        attempt, built = 0, False
        for attempt in range(12):
            cfg = cfg_for(attempt)
            table = bht.HashTable(cfg, local)
            built = table.insert(d_keys, d_vals).success
            if built:
                break
            table.close()
        else:
            table = bht.HashTable(cfg, local)
        wl["build_attempt"], wl["build_success"] = attempt, bool(built)

        def step(timers=None):
            e = [ev() for _ in range(4)] if timers is not None else None
            if e: e[0].record(stream)
            table.clear()
            if e: e[1].record(stream)
            table.insert(d_keys, d_vals, want_result=False)
            if e: e[2].record(stream)
            table.find(d_pos, d_out)
            if e: e[3].record(stream)
            if timers is not None:
                timers.append(e)

        for _ in range(max(args.warmup, 3)):
            step()
        outcome = table.last_insert_result()
        built = built and outcome.success  # a cell at the edge of what the table holds may build one time and not the next
        barrier()
        launches0 = bht.kernel_launch_count()
        sampler.start()
        timers = []
        t_start, t_end = ev(), ev()
        t_start.record(stream)
        for _ in range(args.steps):
            step(timers)
        t_end.record(stream)
        sampler.sample_until(t_end)
        barrier()
        clocks = sampler.stop()
        launches = bht.kernel_launch_count() - launches0
        total_ms = t_start.elapsed_time(t_end)
        ms_step = total_ms / args.steps
        clear_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in timers]))
        ins_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in timers]))
        find_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in timers]))
        value = 2 * n / (ms_step * 1e-3) / 1e6

        # probe counts of this very workload (device counters = probe_stats, probe_stats.hpp:12-31)
        outcome = table.last_insert_result()
        _, fs100 = table.find(d_pos, d_out, want_stats=True)
        assert fs100.hits == outcome.inserted  # every stored pair is found (all n of them when the build succeeded)
        built = built and outcome.success
        if outcome.success:
            checksum_ok = fs100.value_sum == int((d_vals.to(torch.int64) & 0xFFFFFFFF).sum().item())
            assert checksum_ok, "find checksum mismatch"

        def timed_find(q):
            torch.cuda.synchronize()
            a, b_ = ev(), ev()
            ts = []
            for _ in range(3):
                a.record(stream)
                table.find(q, d_out)
                b_.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b_))
            return float(np.mean(ts))
        f50_ms = timed_find(d_mixed)
        f0_ms = timed_find(d_abs)
        _, fs50 = table.find(d_mixed, d_out, want_stats=True)
        _, fs0 = table.find(d_abs, d_out, want_stats=True)
        assert fs0.hits == 0 and (not outcome.success or fs50.hits == int(round(0.5 * n)))

        # the insert op = partition passes + region build (shared-memory-blocked build) + the bulk-insert kernel that
        # finishes the eviction walks: split at the launch of that kernel (events inside the library)
        prep, probe = [], []
        for _ in range(5):
            table.clear()
            table.insert(d_keys, d_vals, want_result=False)
            a_ms, b_ms = table.last_insert_phases()
            prep.append(a_ms)
            probe.append(b_ms)
        table.find(d_keys, d_out)
        ins_prepare_ms, ins_kernel_ms = float(np.mean(prep)), float(np.mean(probe))

        # the reference's own call shape, build(keys, cfg): values = value_for_key(key), made inside the first pass
        def timed_keys_only_build():
            ts = []
            a, b_ = ev(), ev()
            for _ in range(5):
                table.clear()
                torch.cuda.synchronize()
                a.record(stream)
                table.insert(d_keys, None, want_result=False)
                b_.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b_))
            return float(np.mean(ts))
        ins_keys_only_ms = timed_keys_only_build()
        table.clear()
        table.insert(d_keys, d_vals, want_result=False)  # back to the explicit pairs for whatever follows

        peaks = load_peaks()
        ins_bytes = bht.predict_sectors(KIND, B, outcome.mean_probes, bht.OP_INSERT) * 32 * n
        find_bytes = bht.predict_sectors(KIND, B, fs100.mean_probes, bht.OP_FIND) * 32 * n
        dom_insert = ins_kernel_ms >= find_ms
        dom_bytes, dom_ms = (ins_bytes, ins_kernel_ms) if dom_insert else (find_bytes, find_ms)
        traffic = load_traffic() if (n == N_KEYS and HEADLINE) else {}
        roof = lambda by, ms, kern=None: {"bound": "hbm", "achieved": by / (ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],  # noqa: E731
                                          "unit": "GB/s", "frac": by / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                          "traffic": traffic.get(kern), "peak_source": peaks["source"]}
        hashes = bht.hash_count(KIND)
        ins_kernel = {"bcht": f"bulk_insert_cuckoo_kernel<{B},3,1>", "1cht": "bulk_insert_cuckoo_kernel<1,4,0>",
                      "bp2ht": "claim_insert_p2_kernel", "iht": "claim_insert_iht_kernel"}[KIND]
        find_kernel = f"bulk_find_kernel<{B},{hashes},{'true' if KIND in ('bcht', '1cht') else 'false'}>"
        dom_kernel = ins_kernel if dom_insert else find_kernel
        roofline = roof(dom_bytes, dom_ms, dom_kernel)
        roofline["kernel"] = dom_kernel
        roofline["algorithmic_bytes_per_key"] = dom_bytes / n
        roofline["frac_of_8TBps"] = dom_bytes / (dom_ms * 1e-3) / 8e12
        # the stricter variant: the sector model plus the streamed arrays (find: 4 B key in + 4 B value out; insert: 8 B in)
        roofline["frac_with_streaming_io"] = (dom_bytes + 8 * n) / (dom_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]
        # the other ceiling of this part: HBM serves ~48.7 G random accesses per second whatever their size up to 128 B
        # (tools/microbench, profiles/r01_microbench_gather_atomics.txt: 128-byte line gathers over 444 MB).  b = 16 is the
        # bucket size at which that rate equals the byte roof; smaller buckets (b = 8: 64 B, 1cht: 8 B) hit the access
        # rate at a fraction of the bytes, which is what their `frac` below 1 means.
        rate_peak = 48.7e9
        dom_probes = (outcome.mean_probes + 1.0 if dom_insert else fs100.mean_probes) * n  # an insert also writes a dirtied sector back
        roofline["access_rate"] = {"bound": "hbm random accesses", "achieved": dom_probes / (dom_ms * 1e-3) / 1e9, "peak": rate_peak / 1e9,
                                   "unit": "G accesses/s", "frac": dom_probes / (dom_ms * 1e-3) / rate_peak,
                                   "peak_source": "profiles/r01_microbench_gather_atomics.txt (random 128 B line gather, 444 MB)"}
        roofline["note"] = ("achieved = sector-model bytes (probes x 4 sectors, + 1 written sector per inserted pair, x 32 B) / "
                            "this kernel's CUDA-event time; traffic = its ncu dram bytes per launch (L2 hits make it smaller "
                            "than the model). detail.roofline_insert_op is the whole bulk insert (partition passes, "
                            "shared-memory region build, eviction-walk kernel) over the DRAM bytes it actually moves")
        detail = {
            "clear_ms": clear_ms, "insert_ms": ins_ms, "find_ms": find_ms,
            "clear_note": "bht_clear defers the fill; the blocked build's region write-back (K11) writes every slot of the store "
                          "once, empty ones included, so the step has no separate fill pass (DESIGN.md, Deferred fill)",
            "insert_blocked_build_ms": ins_prepare_ms, "insert_walk_kernel_ms": ins_kernel_ms,
            "insert_keys_only_ms": ins_keys_only_ms, "insert_keys_only_mkeys": n / (ins_keys_only_ms * 1e-3) / 1e6,
            "insert_mkeys": n / ins_ms / 1e3, "find_100_mkeys": n / find_ms / 1e3,
            "find_50_mkeys": n / f50_ms / 1e3, "find_0_mkeys": n / f0_ms / 1e3,
            "insert_probes_per_key": outcome.mean_probes, "find_100_probes_per_key": fs100.mean_probes,
            "find_50_probes_per_key": fs50.mean_probes, "find_0_probes_per_key": fs0.mean_probes,
            "roofline_insert_op": insert_op_roofline(ins_bytes, ins_ms, traffic.get("insert_op"), peaks),
            "roofline_find_100": roof(find_bytes, find_ms, find_kernel),
            "roofline_find_50": roof(bht.predict_sectors(KIND, B, fs50.mean_probes, bht.OP_FIND) * 32 * n, f50_ms),
            "roofline_find_0": roof(bht.predict_sectors(KIND, B, fs0.mean_probes, bht.OP_FIND) * 32 * n, f0_ms),
        }

        # ---- e2e: the same pass through the C ABI with HOST buffers (pinned), copies inside the timed region
        h_keys = d_keys.cpu().pin_memory()
        h_vals = d_vals.cpu().pin_memory()
        h_out = torch.empty(n, dtype=torch.int32).pin_memory()
        e2e_steps = max(2, min(args.steps, 5))

        def e2e_leg(values):
            def e2e_step():
                table.clear()
                table.insert(h_keys, values, want_result=False)  # returns when the host arrays have crossed PCIe; the rest of
                table.find(h_keys, h_out)                        # the build runs under the first query chunks' H2D copies
                return table.last_insert_result()                # the step's result read back (D2H), after the answers
            e2e_step()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                o = e2e_step()
            torch.cuda.synchronize()
            return o, (time.perf_counter() - t0) / e2e_steps

        # (1) the reference's own call: build(keys, cfg) pairs key k with value_for_key(k) (table.cpp:234) - keys only
        # cross PCIe, the values are made on the device; (2) explicit (key, value) pairs, as the device-resident leg
        o, e2e_s = e2e_leg(None)
        want = bht.values_for_keys(d_keys.view(torch.int32)).cpu()
        assert not o.success or torch.equal(h_out, want.view(torch.int32))
        built = built and o.success
        o, e2e_pairs_s = e2e_leg(h_vals)
        assert not o.success or torch.equal(h_out, h_vals)
        wl["build_success"] = bool(built and o.success)  # every build of the run, timed ones included
        e2e = {"value": 2 * n / e2e_s / 1e6, "unit": "MKeys/s", "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 4 * n + 64, "ms_per_step": e2e_s * 1e3,
               "api": "bht_insert(keys, NULL = value_for_key, BHT_MEM_HOST, result = NULL) / bht_find(BHT_MEM_HOST) / "
                      "bht_last_insert_result: the reference's build(keys, cfg) + find_key loop on pinned host arrays; the "
                      "insert returns when its chunks have crossed PCIe (each fed to the blocked build's first pass as it "
                      "lands), the rest of the build runs under the first query chunks",
               "explicit_values": {"value": 2 * n / e2e_pairs_s / 1e6, "unit": "MKeys/s", "h2d_bytes_per_step": 12 * n,
                                   "d2h_bytes_per_step": 4 * n + 64, "ms_per_step": e2e_pairs_s * 1e3,
                                   "api": "bht_insert(keys, values, BHT_MEM_HOST) / bht_find(BHT_MEM_HOST)"}}

        cpu = cpu_baseline_leg(args, present, n) if not (args.no_cpu_baseline or args.device_keys) else None
        line = {
            "metric": METRIC, "value": value, "unit": "MKeys/s", "n_gpus": 1, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32/u64 integer", "data": ("synthetic: unique u32 keys from the device bijection" if args.device_keys
                                                    else data_label(args)),
            "config": wl, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "detail": detail,
        }
        print(json.dumps(line), flush=True)
        return 0

    # ---- the sharded table (N > 1, or --sharded on one GPU): keys generated on the device, routing inside the timed region
    if world == 1 and not dist.is_initialized():
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        with StdoutToStderr():
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=device)
    keys, vals = bht.generate_unique_keys(SEED, rank * n, n, device=local)
    keys, vals = keys.view(torch.int32), vals.view(torch.int32)
    sharded = bht.ShardedTable(cfg, device=local, chunk=args.chunk)
    out = torch.empty(n, dtype=torch.int32, device=device)
    table = sharded.ops.table

    def step(marks=None):
        if marks is not None: marks.append(ev()); marks[-1].record(stream)
        table.clear()
        o = sharded.insert(keys, vals)  # one host read at the end: the aggregated outcome (and the overflow flag)
        if marks is not None: marks.append(ev()); marks[-1].record(stream)
        sharded.find(keys, out)
        if marks is not None: marks.append(ev()); marks[-1].record(stream)
        return o

    with StdoutToStderr():
        for _ in range(max(args.warmup, 3)):
            o = step()
    assert o.success, o
    assert torch.equal(out, vals), "sharded find answers differ from the inserted values"
    barrier()
    launches0 = bht.kernel_launch_count()
    sampler.start()
    marks_all = []
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    for _ in range(args.steps):
        marks = []
        step(marks)
        marks_all.append(marks)
    t_end.record(stream)
    sampler.sample_until(t_end)
    barrier()
    clocks = sampler.stop()
    ms_step = max_over_ranks(t_start.elapsed_time(t_end) / args.steps)
    ins_ms = max_over_ranks(float(np.mean([m[0].elapsed_time(m[1]) for m in marks_all])))
    find_ms = max_over_ranks(float(np.mean([m[1].elapsed_time(m[2]) for m in marks_all])))
    launches = bht.kernel_launch_count() - launches0

    # the shard's own work without any routing: the same n pairs straight into this rank's table (HBM part of the step)
    local_ms = []
    for _ in range(3):
        table.clear()
        torch.cuda.synchronize()
        a, b_ = ev(), ev()
        a.record(stream)
        table.insert(keys, vals, want_result=False)
        table.find(keys, out)
        b_.record(stream)
        torch.cuda.synchronize()
        local_ms.append(a.elapsed_time(b_))
    local_ms = max_over_ranks(float(np.mean(local_ms)))
    local_outcome = table.last_insert_result()
    _, fs = table.find(keys, out, want_stats=True)
    # the exchange alone: the all-to-alls of one step (keys + values out, queries out, answers back), equal splits
    cap = sharded.segment_cap(min(n, args.chunk))
    n_chunks = -(-n // args.chunk)
    sendbuf, recvbuf = torch.empty(world * cap, dtype=torch.int32, device=device), torch.empty(world * cap, dtype=torch.int32, device=device)
    a2a_ms = []
    for _ in range(3):
        torch.cuda.synchronize()
        a, b_ = ev(), ev()
        a.record(stream)
        for _c in range(n_chunks * 4):
            dist.all_to_all_single(recvbuf, sendbuf)
        b_.record(stream)
        torch.cuda.synchronize()
        a2a_ms.append(a.elapsed_time(b_))
    a2a_ms = max_over_ranks(float(np.mean(a2a_ms)))
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and n <= 100_000_000:
        cpu = cpu_baseline_leg(args, keys.cpu().numpy().view(np.uint32), n)
    barrier()  # the other ranks wait for rank 0's CPU leg before the group is torn down
    if world == 1:
        wl["parallelism"] = "the sharded path with a world of one (no routing: one shard owns every key)"
    if rank == 0:
        value = 2 * n * world / (ms_step * 1e-3) / 1e6
        peaks = load_peaks()
        alg_bytes = (bht.predict_sectors(KIND, B, local_outcome.mean_probes, bht.OP_INSERT) +
                     bht.predict_sectors(KIND, B, fs.mean_probes, bht.OP_FIND)) * 32 * n  # per GPU per step
        nvlink_peak = 900.0  # GB/s per direction per GPU (NVLink 5 through NVSwitch)
        # bytes one GPU sends (= receives) per step: (G-1)/G of its pairs (8 B), of its queries (4 B) and of the answers (4 B)
        nv_bytes = n * (world - 1) / world * 16.0
        padded = n_chunks * 4 * (world - 1) * cap * 4.0  # what the fixed-segment exchange actually moves per GPU each way
        roofline = {
            "bound": "hbm", "achieved": alg_bytes / (ms_step * 1e-3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": alg_bytes / (ms_step * 1e-3) / 1e9 / peaks["hbm_gbs"], "traffic": None, "peak_source": peaks["source"],
            "kernel": "whole sharded step per GPU: K8 partition, all-to-all, chunked blocked build, bulk find, all-to-all back, K9",
            "algorithmic_bytes_per_key": alg_bytes / (2 * n),
            "frac_local_only": alg_bytes / (local_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "nvlink": {"bound": "nvlink all-to-all", "bytes_per_gpu_per_step_each_way": nv_bytes, "padded_bytes": padded,
                       "achieved": nv_bytes / (ms_step * 1e-3) / 1e9, "peak": nvlink_peak, "unit": "GB/s",
                       "frac": nv_bytes / (ms_step * 1e-3) / 1e9 / nvlink_peak,
                       "alltoall_only_ms": a2a_ms,
                       "alltoall_only_frac": (padded / (a2a_ms * 1e-3) / 1e9 / nvlink_peak) if world > 1 else None,
                       "note": "frac = routed bytes / whole step time / 900 GB/s: how far the step is from being bound by the "
                               "exchange; alltoall_only = the step's all-to-alls issued back to back with nothing else"},
            "note": "achieved = sector-model bytes of this GPU's build + find / the whole step (routing included); "
                    "frac_local_only = the same bytes / the same pairs inserted and found without routing",
        }
        line = {
            "metric": METRIC, "value": value, "unit": "MKeys/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32/u64 integer",
            "data": "synthetic: unique u32 keys from a device-side bijection of a counter",
            "config": wl, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "MKeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 128,
                    "note": "sharded pass: inputs are device-resident per rank (the key space of a 4-billion-key table does not "
                            "come from one host); routing (NCCL all-to-all) and the outcome read-back are inside"},
            "gpu_launches": int(launches), "clocks": clocks,
            "detail": {"insert_ms": ins_ms, "find_ms": find_ms, "local_build_find_ms": local_ms, "alltoall_only_ms": a2a_ms,
                       "chunk": args.chunk, "segment_cap": cap, "chunks_per_call": n_chunks,
                       "insert_mkeys": n * world / ins_ms / 1e3, "find_mkeys": n * world / find_ms / 1e3,
                       "insert_probes_per_key": local_outcome.mean_probes, "find_probes_per_key": fs.mean_probes,
                       "exchange": "fixed segments, equal-split all_to_all_single, device-side counts; host reads per call: 1"},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def insert_op_roofline(model_bytes, ms, traffic, peaks):
    """The whole bulk insert against the HBM roof ON ITS OWN BYTES: a blocked build moves far fewer DRAM bytes than the
    random-sector model charges (three streaming passes + the walks instead of one random line per probe), so dividing
    the model's bytes by its time says nothing about how close it is to the hardware (round 1 printed 1.31 there)."""
    achieved = traffic / (ms * 1e-3) / 1e9 if traffic else None
    return {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"] if achieved else None, "traffic": traffic,
            "sector_model_bytes": model_bytes, "peak_source": peaks["source"],
            "note": "achieved = measured DRAM bytes of the insert's launches (ncu, profiles/traffic.json) / its CUDA-event time; "
                    "null when no capture of these kernel sources is committed"}


def load_traffic():
    """DRAM bytes per launch of the two hot kernels from the committed `ncu --set full` capture of this very
    workload (tools/ncu_summary.py --traffic-json); None when no capture has been committed."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        data = json.load(open(path))
        if data.get("_csrc_sha") == csrc_stamp():  # captured from these very kernel sources (tools/gpu_round.sh ncu)
            return data
    return {}


def load_peaks():
    """HBM peak for the roofline: the driver-written MEASURED_PEAKS.json when present (whatever it calls the HBM copy
    bandwidth; the burst figure when it distinguishes, because every kernel here is timed alone by its own CUDA events),
    else the profiling recipe's fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        flat = {}

        def walk(prefix, node):
            if isinstance(node, dict):
                for k, v in node.items():
                    walk(f"{prefix}.{k}" if prefix else str(k), v)
            elif isinstance(node, (int, float)) and not isinstance(node, bool):
                flat[prefix.lower()] = float(node)
        walk("", p)
        hbm = {k: v for k, v in flat.items() if "hbm" in k and ("gb" in k or "bw" in k or "bandwidth" in k or "copy" in k)}
        if hbm:
            key = next((k for k in hbm if "burst" in k), None) or ("hbm_gbs" if "hbm_gbs" in hbm else sorted(hbm)[0])
            value = hbm[key]
            if value > 100000:  # bytes/s rather than GB/s
                value /= 1e9
            if 1000.0 < value < 20000.0:
                return {"hbm_gbs": value, "source": f"MEASURED_PEAKS.json ({key})"}
    except (OSError, ValueError):
        pass
    return {"hbm_gbs": 6650.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)"}


def cpu_baseline_leg(args, present, n):
    """The reference CPU implementation timed on this box's host cores, bounded to roughly 10-30 s."""
    from oracle import binding
    if not binding.ref_available():
        return {"value": None, "unit": "MKeys/s", "cores": 0, "kind": "reference", "sample": "oracle/_ref not built"}
    ref = binding.ref()
    threads = ref.hardware_concurrency()
    ocfg = make_ref_config(ref, n)
    probe_n = min(n, 1_000_000)
    tb, tf, _, _ = cpu_reference_pass(ref, ocfg, present, present, probe_n, threads)
    rate = 2 * probe_n / max(tb + tf, 1e-9)
    n_sample = int(min(n, max(1_000_000, rate * 20.0 / 2)))
    tb, tf, out, hits = cpu_reference_pass(ref, ocfg, present, present, n_sample, threads)
    assert out["success"] and hits == n_sample
    return {"value": 2 * n_sample / (tb + tf) / 1e6, "unit": "MKeys/s", "cores": threads, "kind": "reference",
            "insert_mkeys": n_sample / tb / 1e6, "find_mkeys": n_sample / tf / 1e6,
            "sample": f"first {n_sample} of the {n} keys: reference build(parallel, {threads} workers) into the "
                      f"full-size table + {n_sample} positive find_key calls over {threads} threads"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--keys", type=int, default=N_KEYS, help="keys per GPU")
    ap.add_argument("--chunk", type=int, default=1 << 24, help="sharded pipeline chunk (keys)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="headline",
                    help="headline (bcht b=16 LF 0.9) | " + " | ".join(k for k in CONFIGS if k != "headline") + " | kind:b:lf[:t]")
    ap.add_argument("--sharded", action="store_true", help="one GPU through the sharded path (a world of one)")
    ap.add_argument("--device-keys", action="store_true", help="generate keys on the device (large --keys)")
    ap.add_argument("--workload", default="reference", choices=["reference", "numpy"],
                    help="reference: the reference harness's generate_keys / generate_queries for seed 1; numpy: MT19937 + unique")
    args = ap.parse_args()
    select_config(args.config)
    if args.impl == "reference":
        return run_reference(args)
    return run_cuda(args)


if __name__ == "__main__":
    sys.exit(main())
