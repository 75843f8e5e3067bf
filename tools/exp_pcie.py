"""PCIe ceiling of the e2e leg: pinned H2D / D2H copy rates on this box and the host-buffer insert / find times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht

n = 50_000_000
h = torch.empty(2 * n, dtype=torch.int32).pin_memory()
d = torch.empty(2 * n, dtype=torch.int32, device="cuda")
s2 = torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h.copy_(d, non_blocking=True))
print(f"H2D 400 MB: {h2d*1e3:.2f} ms = {0.4/h2d:.1f} GB/s;  D2H 400 MB: {d2h*1e3:.2f} ms = {0.4/d2h:.1f} GB/s")
h_b = torch.empty(n, dtype=torch.int32).pin_memory(); d_b = torch.empty(n, dtype=torch.int32, device="cuda")
def both():
    d[:n].copy_(h[:n], non_blocking=True)
    with torch.cuda.stream(s2):
        h_b.copy_(d_b, non_blocking=True)
bt = t(both)
print(f"H2D 200 MB || D2H 200 MB: {bt*1e3:.2f} ms")

cfg = bht.make_config("bcht", n, 0.9, 16, seed=bht.mix_seed(1, 0x100))
k, v = bht.generate_unique_keys(1, 0, n, device=0)
hk, hv = k.view(torch.int32).cpu().pin_memory(), v.view(torch.int32).cpu().pin_memory()
ho = torch.empty(n, dtype=torch.int32).pin_memory()
table = bht.HashTable(cfg, 0)
def ins(): table.clear(); table.insert(hk, hv)
def ins_nores(): table.clear(); table.insert(hk, hv, want_result=False)
def fnd(): table.find(hk, ho)
print(f"host insert (with result): {t(ins)*1e3:.2f} ms; without result {t(ins_nores)*1e3:.2f} ms; host find {t(fnd)*1e3:.2f} ms; floor = {(0.4/ (0.4/h2d) + 0.2/(0.4/h2d))*1e3:.2f} ms")
assert torch.equal(ho, hv)
# keys-only build (values = NULL -> value_for_key on the device): half the H2D bytes of the insert
want = bht.values_for_keys(k.view(torch.int32)).view(torch.int32).cpu()
def ins_keys(): table.clear(); table.insert(hk)
def ins_keys_nores(): table.clear(); table.insert(hk, want_result=False)
def both_legs(): table.clear(); table.insert(hk); table.find(hk, ho)
print(f"keys-only host insert (with result): {t(ins_keys)*1e3:.2f} ms; without result {t(ins_keys_nores)*1e3:.2f} ms; "
      f"insert + find {t(both_legs)*1e3:.2f} ms; floor = {(0.2 / (0.4/h2d) + 0.2/(0.4/h2d))*1e3:.2f} ms")
assert torch.equal(ho, want)
