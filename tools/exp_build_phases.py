"""Blocked build A/B: timing (CUDA events, warm) + full check of one build.  python tools/exp_build_phases.py [n] [kind b lf]
BHT_B200_LIB selects the library build (csrc/Makefile VARIANT=...)."""
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
if kind != "bcht":
    table.set_blocked_insert(3)
ts, prep, walk = [], [], []
for i in range(8):
    table.clear(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); table.insert(k, v, want_result=False); e1.record(); torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
        a, c = table.last_insert_phases(); prep.append(a); walk.append(c)
o = table.last_insert_result()
ok = torch.equal(table.find(k).view(torch.int32), v) and table.occupied_slots() == n and table.count_inadmissible() == 0
m = lambda x: sum(x) / len(x)
print(f"{os.environ.get('BHT_B200_LIB', 'default')[-24:]:24s} {kind} b={b} lf={lf} n={n}: insert {m(ts):.3f} ms (min {min(ts):.3f}) = {n/m(ts)/1e3:.0f} MKeys/s; "
      f"passes {m(prep):.3f} walk {m(walk):.3f}; probes {o.mean_probes:.4f} ok={o.success} check={ok}", flush=True)
