"""A table that FITS the 126 MB L2 (bcht b=16, 11.25 M keys at load factor 0.9 = 100 MB of slots) next to the 444 MB
headline table: general-kernel build (caller order) + positive / negative finds, timed, for the ncu comparison of L2 hit
rate, DRAM bytes and atomic throughput L2-resident vs HBM-resident.
    python tools/exp_l2_resident.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht

n = int(sys.argv[1]) if len(sys.argv) > 1 else 11_250_000
cfg = bht.make_config("bcht", n, 0.9, 16, seed=bht.mix_seed(1, 0x100))
k, v = bht.generate_unique_keys(1, 0, n, device=0)
a = bht.generate_unique_keys(1, n, n, device=0, with_values=False)
k, v, a = k.view(torch.int32), v.view(torch.int32), a.view(torch.int32)
table = bht.HashTable(cfg, 0)
table.set_blocked_insert(0)  # the per-bucket kernel: bucket read + 64-bit CAS per pair, the paper's insert
out = torch.empty(n, dtype=torch.int32, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
ti, tf, tn = [], [], []
for i in range(6):
    table.clear(); torch.cuda.synchronize()
    e = [ev() for _ in range(4)]
    e[0].record(); table.insert(k, v, want_result=False); e[1].record(); table.find(k, out); e[2].record(); table.find(a, out); e[3].record()
    torch.cuda.synchronize()
    if i >= 2:
        ti.append(e[0].elapsed_time(e[1])); tf.append(e[1].elapsed_time(e[2])); tn.append(e[2].elapsed_time(e[3]))
o = table.last_insert_result()
m = lambda x: sum(x) / len(x)
print(f"bcht b=16 n={n} table {cfg.capacity * 8 / 1e6:.0f} MB ok={o.success}: insert (caller order) {n / m(ti) / 1e3:.0f} MKeys/s, "
      f"find 100% {n / m(tf) / 1e3:.0f} MKeys/s, find 0% {n / m(tn) / 1e3:.0f} MKeys/s; probes/insert {o.mean_probes:.4f}")
