"""Does an HBM-saturating probe kernel slow the PCIe copies that run beside it?  H2D / D2H of 200 MB alone, and while bulk
finds (or caller-order bulk inserts) over a 444 MB table run back to back on another stream.  python tools/exp_pcie_contention.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht

n = 50_000_000
cfg = bht.make_config("bcht", n, 0.9, 16, seed=bht.mix_seed(1, 0x100))
k, v = bht.generate_unique_keys(1, 0, n, device=0)
k, v = k.view(torch.int32), v.view(torch.int32)
table = bht.HashTable(cfg, 0)
table.insert(k, v)
out = torch.empty_like(k)
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
side = torch.cuda.Stream()

def copy_ms(fn, busy):
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        if busy is not None:
            with torch.cuda.stream(side):
                for _ in range(8):
                    busy(side)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)

t2 = bht.HashTable(cfg, 0)
t2.set_blocked_insert(0)
def finds(s): table.find(k, out, stream=s)
def inserts(s):
    t2.clear(stream=s)
    t2.insert(k, v, want_result=False, stream=s)
for name, busy in [("alone", None), ("beside bulk finds", finds), ("beside caller-order bulk inserts", inserts)]:
    try:
        up = copy_ms(lambda: d.copy_(h, non_blocking=True), busy)
        down = copy_ms(lambda: h.copy_(d, non_blocking=True), busy)
        print(f"{name:34s}: H2D 200 MB {up:.2f} ms = {0.2 / up * 1e3:.1f} GB/s;  D2H 200 MB {down:.2f} ms = {0.2 / down * 1e3:.1f} GB/s", flush=True)
    except TypeError as e:
        print(name, "skipped:", e)
