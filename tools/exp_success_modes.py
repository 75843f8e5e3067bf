"""Build success of bcht b=16 at a high load factor per bulk-build schedule (caller order / L2-routed / smem-blocked)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht
from paper_2108_07232_b200 import workload

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
lf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.99
trials = int(sys.argv[3]) if len(sys.argv) > 3 else 30
keys = workload.generate_keys(bht.mix_seed(1, 0x6B657973), n, device=0).keys.view(torch.int32)
vals = bht.values_for_keys(keys)
for mode, label, env in ((0, "caller order, direct engine", {"BHT_DIRECT": "1"}), (0, "caller order, staged engine", {"BHT_DIRECT": "0"}),
                         (2, "L2-routed", {"BHT_DIRECT": "1"}), (3, "smem-blocked", {"BHT_DIRECT": "1"})):
    os.environ.update(env)
    ok, dropped, probes = 0, [], 0.0
    for t in range(trials):
        cfg = bht.make_config("bcht", n, lf, 16, seed=bht.mix_seed(1234, t))
        table = bht.HashTable(cfg, 0)
        table.set_blocked_insert(mode)
        o = table.insert(keys, vals)
        ok += o.success
        probes += o.mean_probes
        if not o.success:
            dropped.append(o.failed)
        table.close()
    print(f"{label:30s} lf={lf} n={n}: {ok}/{trials} builds succeed, mean probes {probes / trials:.4f}, dropped per failed build {dropped[:12]}", flush=True)
