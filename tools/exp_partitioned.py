"""Experiment: how fast are bulk insert / find when the keys arrive grouped by the table region of their first
bucket (P contiguous regions)?  Tells whether an L2-blocked build is worth building into the library."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2108_07232_b200 as bht
from bench import make_workload

n = 50_000_000
present, absent, values = make_workload(n, 1)
cfg = bht.make_config("bcht", n, 0.9, 16, seed=bht.mix_seed(1, 0x100))
dev = torch.device("cuda:0")
k = torch.from_numpy(present.view(np.int32)).to(dev)
v = torch.from_numpy(values.view(np.int32)).to(dev)
a, b, r = cfg.hashes[0]
h0 = bht.hash_keys(a, b, r, k).view(torch.int32).long()
table = bht.HashTable(cfg, 0)
table.set_blocked_insert(False)  # the input is grouped here, not by the library
out = torch.empty(n, dtype=torch.int32, device=dev)

def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        table.clear(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)

for P in ([int(x) for x in sys.argv[1:]] or [1, 2, 4, 8, 16, 32, 64]):
    if P == 1:
        kk, vv = k, v
    else:
        part = (h0 * P) // cfg.num_buckets
        order = torch.argsort(part, stable=True)
        kk, vv = k[order].contiguous(), v[order].contiguous()
    t_ins = timed(lambda: table.insert(kk, vv, want_result=False))
    o = table.last_insert_result()
    table.clear(); table.insert(kk, vv, want_result=False)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); table.find(kk, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"P={P:3d} insert {t_ins:.3f} ms = {n/t_ins/1e3:8.0f} MKeys/s (probes {o.mean_probes:.4f}, ok={o.success})   find {min(ts):.3f} ms = {n/min(ts)/1e3:8.0f} MKeys/s", flush=True)
