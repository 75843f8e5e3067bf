"""Build success of bcht b=16 at a high load factor against the number of keys in flight (BHT_INSERT_CTAS)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht
from paper_2108_07232_b200 import workload

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
lf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.99
trials = int(sys.argv[3]) if len(sys.argv) > 3 else 60
keys = workload.generate_keys(bht.mix_seed(1, 0x6B657973), n, device=0).keys.view(torch.int32)
vals = bht.values_for_keys(keys)
for ctas in ("0", "148", "16", "1"):
    os.environ["BHT_INSERT_GRID"] = ctas; bht.reload_tuning()
    ok, dropped = 0, 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    for t in range(trials):
        cfg = bht.make_config("bcht", n, lf, 16, seed=bht.mix_seed(1234, t))
        table = bht.HashTable(cfg, 0)
        table.set_blocked_insert(0)
        ev0.record(); table.insert(keys, vals, want_result=False); ev1.record(); ev1.synchronize()
        ms += ev0.elapsed_time(ev1)
        o = table.last_insert_result()
        ok += o.success
        dropped += o.failed
        table.close()
    print(f"grid={ctas or 'full':>4s} lf={lf} n={n}: {ok}/{trials} builds succeed, {dropped} pairs dropped in total, "
          f"{ms / trials:.3f} ms per build", flush=True)
