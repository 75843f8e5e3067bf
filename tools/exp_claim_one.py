"""One bp2ht / iht bulk build of n pairs (for ncu): python tools/exp_claim_one.py [kind] [n] [mode]
mode 3 = counter-claimed kernels (csrc/insert_claim.cu), mode 0 = bucket-reading kernels (insert_p2.cu / insert_iht.cu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht
kind = sys.argv[1] if len(sys.argv) > 1 else "bp2ht"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50_000_000
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 3
extra = {"threshold": 12} if kind == "iht" else {}
cfg = bht.make_config(kind, n, 0.8, 16, seed=bht.mix_seed(1, 0x100), **extra)
k, v = bht.generate_unique_keys(1, 0, n, device=0)
k, v = k.view(torch.int32), v.view(torch.int32)
table = bht.HashTable(cfg, 0)
table.set_blocked_insert(mode)
for _ in range(3):
    table.clear()
    table.insert(k, v, want_result=False)
torch.cuda.synchronize()
print(kind, mode, table.last_insert_result())
