#!/usr/bin/env python
"""Summarise an .ncu-rep (one `ncu --set full` capture) into the counters DESIGN.md argues with.

    python tools/ncu_summary.py gpurun_out/r01d/prof_find.ncu-rep [--out profiles/r01_find.txt]
"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_op_atom.sum",
    "lts__t_sectors_op_red.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ldgsts.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ldgsts.sum",
    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum", "l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum",
    "lts__t_sectors_op_atom.sum.per_second", "lts__t_requests_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__warps_eligible.avg.per_cycle_active",
    "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
]
PREFIX = ["smsp__average_warps_issue_stalled", "smsp__average_warp_latency_issue_stalled"]


def main():
    rep = sys.argv[1]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"== {name[:110]}")
        for i, h in enumerate(hdr):
            v = r[i]
            keep = h in WANT
            if not keep and any(h.startswith(p) for p in PREFIX) and "not_issued" not in h:
                try:
                    keep = float(v.replace(",", "")) >= 0.3
                except ValueError:
                    keep = False
            if keep:
                lines.append(f"{h:82s} {v:>18s} {units[i]}")
    if "--traffic-json" in sys.argv:  # merge dram bytes per launch into profiles/traffic.json (read by bench.py)
        import json, os, re
        path = sys.argv[sys.argv.index("--traffic-json") + 1]
        data = json.load(open(path)) if os.path.exists(path) else {}
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            m = re.match(r"(?:void )?(?:bht_b200::)?(\w+)<([^>]*)>", name)
            plain = re.search(r"(\w+_kernel)\(", name)  # untemplated kernels of an anonymous namespace: "unnamed>::name(args)"
            key = (f"{m.group(1)}<{m.group(2).replace(' ', '').replace('(int)', '').replace('(bool)', '')}>" if m
                   else (plain.group(1) if plain else name))
            key = key.replace(",1>", ",true>").replace(",0>", ",false>") if key.startswith("bulk_find") else key

            def val(metric):
                v = float(r[hdr.index(metric)].replace(",", ""))
                u = units[hdr.index(metric)]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            data[key] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        parts = [k for k in data if k.split("<")[0] in ("group_scatter_kernel", "bin_split_kernel", "region_build_kernel",
                                                        "bulk_insert_cuckoo_kernel")]
        if len(parts) == 4:  # the whole bulk insert of the blocked build: its four launches
            data["insert_op"] = sum(data[k] for k in parts)
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        data["_csrc_sha"] = bench.csrc_stamp()  # bench.py quotes these numbers only for the sources they were measured on
        json.dump(data, open(path, "w"), indent=1)
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(f"# ncu --set full --clock-control none summary of {rep}\n" + text)
    print(text)


if __name__ == "__main__":
    main()
