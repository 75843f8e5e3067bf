"""One shared-memory-blocked build (for ncu): python tools/exp_smem_one.py [n] [mode]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = bht.make_config("bcht", n, 0.9, 16, seed=bht.mix_seed(1, 0x100))
k, v = bht.generate_unique_keys(1, 0, n, device=0)
k, v = k.view(torch.int32), v.view(torch.int32)
table = bht.HashTable(cfg, 0)
table.set_blocked_insert(mode)
for _ in range(3):
    table.clear()
    table.insert(k, v, want_result=False)
torch.cuda.synchronize()
print(table.last_insert_result())
