"""One routed 50 M-key BCHT build (for ncu captures): region size / CTAs from BHT_REGION_MB / BHT_BLOCKED_CTAS."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht
n = 50_000_000
cfg = bht.make_config("bcht", n, 0.9, 16, seed=bht.mix_seed(1, 0x100))
k, v = bht.generate_unique_keys(1, 0, n, device=0)
k, v = k.view(torch.int32), v.view(torch.int32)
table = bht.HashTable(cfg, 0)
for _ in range(4):
    table.clear(); table.insert(k, v, want_result=False)
torch.cuda.synchronize()
print(table.last_insert_result())
