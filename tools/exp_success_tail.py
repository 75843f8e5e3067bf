"""Build success of bcht b=16 at LF 0.99 when only the LAST part of the batch is inserted with few keys in flight."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht
from paper_2108_07232_b200 import workload

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
lf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.99
trials = int(sys.argv[3]) if len(sys.argv) > 3 else 40
keys = workload.generate_keys(bht.mix_seed(1, 0x6B657973), n, device=0).keys.view(torch.int32)
vals = bht.values_for_keys(keys)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for tail_frac, grid in ((0.0, "0"), (0.005, "1"), (0.02, "1"), (0.02, "16"), (0.05, "16"), (0.1, "16"), (0.1, "64"), (0.3, "64")):
    k1 = int(n * (1 - tail_frac))
    ok, dropped, ms = 0, 0, 0.0
    for t in range(trials):
        cfg = bht.make_config("bcht", n, lf, 16, seed=bht.mix_seed(1234, t))
        table = bht.HashTable(cfg, 0)
        table.set_blocked_insert(0)
        os.environ["BHT_INSERT_GRID"] = "0"; bht.reload_tuning()
        ev0.record()
        o1 = table.insert(keys[:k1], vals[:k1])
        failed = o1.failed
        if k1 < n:
            os.environ["BHT_INSERT_GRID"] = grid; bht.reload_tuning()
            failed += table.insert(keys[k1:], vals[k1:]).failed
        ev1.record(); ev1.synchronize()
        ms += ev0.elapsed_time(ev1)
        ok += failed == 0
        dropped += failed
        table.close()
    print(f"last {tail_frac:5.1%} at grid={grid:>3s}: {ok}/{trials} builds succeed, {dropped} dropped, {ms / trials:.2f} ms per build", flush=True)
