"""Experiment: bulk insert of randomly ordered keys — caller order vs the L2-routed build vs the shared-memory-blocked
build (build_blocked.cu), with a full check of every build."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
kind, b, lf = (sys.argv[2], int(sys.argv[3]), float(sys.argv[4])) if len(sys.argv) > 4 else ("bcht", 16, 0.9)
cfg = bht.make_config(kind, n, lf, b, seed=bht.mix_seed(1, 0x100))
k, v = bht.generate_unique_keys(1, 0, n, device=0)
k, v = k.view(torch.int32), v.view(torch.int32)
table = bht.HashTable(cfg, 0)


def run(label):
    ts = []
    for _ in range(4):
        table.clear(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); table.insert(k, v, want_result=False); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    o = table.last_insert_result()
    ok = torch.equal(table.find(k).view(torch.int32), v) and table.occupied_slots() == n and table.count_inadmissible() == 0
    print(f"{label:34s} insert {min(ts):7.3f} ms = {n/min(ts)/1e3:8.0f} MKeys/s probes {o.mean_probes:.4f} ok={o.success} check={ok}", flush=True)


for mode, label in ((0, "caller order"), (2, "L2-routed"), (3, "smem-blocked"), (1, "auto")):
    table.set_blocked_insert(mode)
    run(label)
