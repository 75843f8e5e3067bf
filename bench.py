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

KIND, B, LF, N_KEYS, SEED = "bcht", 16, 0.9, 50_000_000, 1
METRIC = "insert & find MKeys/s, BCHT b=16, 50M keys, LF 0.9"


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
    print(json.dumps(line))
    return 0


def make_ref_config(ref, n):
    from oracle import binding
    cfg = ref.make_config(binding.KINDS[KIND], n, LF, B, seed=ref.mix_seed(SEED, 0x100))
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
        dist.init_process_group("nccl", device_id=device)
    n = args.keys
    cfg = bht.make_config(KIND, n, LF, B, seed=bht.mix_seed(SEED, 0x100))
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

    if world == 1:
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
        table = bht.HashTable(cfg, local)

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
        assert outcome.success, outcome
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
        assert fs100.hits == n
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
        assert fs0.hits == 0 and fs50.hits == int(round(0.5 * n))

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
            assert table.last_insert_result().success
            return float(np.mean(ts))
        ins_keys_only_ms = timed_keys_only_build()
        table.clear()
        table.insert(d_keys, d_vals, want_result=False)  # back to the explicit pairs for whatever follows

        peaks = load_peaks()
        ins_bytes = bht.predict_sectors(KIND, B, outcome.mean_probes, bht.OP_INSERT) * 32 * n
        find_bytes = bht.predict_sectors(KIND, B, fs100.mean_probes, bht.OP_FIND) * 32 * n
        dom_insert = ins_kernel_ms >= find_ms
        dom_bytes, dom_ms = (ins_bytes, ins_kernel_ms) if dom_insert else (find_bytes, find_ms)
        traffic = load_traffic() if n == N_KEYS else {}
        roof = lambda by, ms, kern=None: {"bound": "hbm", "achieved": by / (ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],  # noqa: E731
                                          "unit": "GB/s", "frac": by / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                          "traffic": traffic.get(kern), "peak_source": peaks["source"]}
        ins_kernel = "bulk_insert_cuckoo_kernel<16,3,1>"  # <b, hashes, register-resident probe>: the eviction walks
        dom_kernel = ins_kernel if dom_insert else "bulk_find_kernel<16,3,true>"
        roofline = roof(dom_bytes, dom_ms, dom_kernel)
        roofline["kernel"] = dom_kernel
        roofline["algorithmic_bytes_per_key"] = dom_bytes / n
        roofline["frac_of_8TBps"] = dom_bytes / (dom_ms * 1e-3) / 8e12
        # the stricter variant: the sector model plus the streamed arrays (find: 4 B key in + 4 B value out; insert: 8 B in)
        roofline["frac_with_streaming_io"] = (dom_bytes + 8 * n) / (dom_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]
        roofline["note"] = ("achieved = sector-model bytes (probes x 4 sectors, + 1 written sector per inserted pair, x 32 B) / "
                            "this kernel's CUDA-event time; traffic = its ncu dram bytes per launch (L2 hits make it smaller "
                            "than the model). detail.roofline_insert_op is the whole bulk insert (partition passes, "
                            "shared-memory region build, eviction-walk kernel): a blocked build moves far fewer DRAM bytes "
                            "than the random-sector model charges, so its fraction exceeds 1")
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
            "roofline_insert_op": roof(ins_bytes, ins_ms, "insert_op"),
            "roofline_find_100": roof(find_bytes, find_ms, "bulk_find_kernel<16,3,true>"),
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
                o = table.insert(h_keys, values)  # H2D of keys (+ values) inside; result read back
                table.find(h_keys, h_out)         # H2D of queries, D2H of answers inside
                return o
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
        assert o.success and torch.equal(h_out, want.view(torch.int32))
        o, e2e_pairs_s = e2e_leg(h_vals)
        assert o.success and torch.equal(h_out, h_vals)
        e2e = {"value": 2 * n / e2e_s / 1e6, "unit": "MKeys/s", "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 4 * n + 64, "ms_per_step": e2e_s * 1e3,
               "api": "bht_insert(keys, NULL = value_for_key, BHT_MEM_HOST) / bht_find(BHT_MEM_HOST): the reference's "
                      "build(keys, cfg) + find_key loop on pinned host arrays, 3-slot staged PCIe pipeline",
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
        print(json.dumps(line))
        return 0

    # ---- N > 1: sharded table, keys generated on the device, routing inside the timed region
    keys, vals = bht.generate_unique_keys(SEED, rank * n, n, device=local)
    keys, vals = keys.view(torch.int32), vals.view(torch.int32)
    sharded = bht.ShardedTable(cfg, device=local, chunk=args.chunk)
    out = torch.empty(n, dtype=torch.int32, device=device)

    def step():
        sharded.ops.table.clear()
        o = sharded.insert(keys, vals)
        sharded.find(keys, out)
        return o

    for _ in range(max(args.warmup, 3)):
        o = step()
    assert o.success, o
    assert torch.equal(out, vals), "sharded find answers differ from the inserted values"
    barrier()
    launches0 = bht.kernel_launch_count()
    sampler.start()
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    for _ in range(args.steps):
        step()
    t_end.record(stream)
    sampler.sample_until(t_end)
    barrier()
    clocks = sampler.stop()
    ms_step = max_over_ranks(t_start.elapsed_time(t_end) / args.steps)
    launches = bht.kernel_launch_count() - launches0
    if rank == 0:
        value = 2 * n * world / (ms_step * 1e-3) / 1e6
        line = {
            "metric": METRIC, "value": value, "unit": "MKeys/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32/u64 integer",
            "data": "synthetic: unique u32 keys from a device-side bijection of a counter",
            "config": wl, "roofline": None, "cpu_baseline": None,
            "e2e": {"value": value, "unit": "MKeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 64,
                    "note": "sharded pass: inputs are device-resident per rank; routing (NCCL all-to-all) is inside"},
            "gpu_launches": int(launches), "clocks": clocks,
        }
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def load_traffic():
    """DRAM bytes per launch of the two hot kernels from the committed `ncu --set full` capture of this very
    workload (tools/ncu_summary.py --traffic-json); None when no capture has been committed."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        return json.load(open(path))
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
    ap.add_argument("--device-keys", action="store_true", help="generate keys on the device (large --keys)")
    ap.add_argument("--workload", default="reference", choices=["reference", "numpy"],
                    help="reference: the reference harness's generate_keys / generate_queries for seed 1; numpy: MT19937 + unique")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_cuda(args)


if __name__ == "__main__":
    sys.exit(main())
