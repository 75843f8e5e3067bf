"""Build success of the bulk build beside the reference's own, same keys and hash constants per seed (under tests/
because the compiled reference is the yardstick; not collected by pytest: run on the GPU box,
`python tests/success_vs_reference.py kind b lf n seeds [threads]`).  For the cuckoo kinds the GPU build is run with the
repair pass on and off."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2108_07232_b200 as bht
from oracle import binding

kind, b, lf, n, seeds = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
ref = binding.ref()
keys_d, _ = bht.generate_unique_keys(7, 0, n, device=0)
keys = keys_d.cpu().numpy().view(np.uint32)
d_keys = keys_d.view(torch.int32)
extra = {"threshold": int(0.8 * b)} if kind == "iht" else {}
ref_ok = on_ok = off_ok = 0
t_ref = 0.0
for s in range(seeds):
    cfg = bht.make_config(kind, n, lf, b, seed=bht.mix_seed(4000 + s, 0x100), **extra)
    t0 = time.time()
    rt, out = ref.build(keys, binding.Config.from_buffer_copy(bytes(cfg)))  # sequential build(), table.cpp:231-238
    t_ref += time.time() - t0
    ref_ok += bool(out["success"])
    rt.close()
    for repair in (True, False):
        t = bht.HashTable(cfg, 0)
        t.set_repair(repair)
        ok = t.insert(d_keys).success
        t.close()
        if repair:
            on_ok += ok
        else:
            off_ok += ok
print(f"{kind} b={b} lf={lf} n={n}: builds that succeed over {seeds} seeds — reference {ref_ok}, bulk build with the repair pass "
      f"{on_ok}, concurrent walks alone {off_ok}  (reference: {t_ref / seeds:.2f} s per build)", flush=True)
