"""Build success and time of bcht b=16 at LF 0.99 against the tail-throttle settings (BHT_TAIL_LF, BHT_TAIL_DIV)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2108_07232_b200 as bht
from paper_2108_07232_b200 import workload

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
lf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.99
trials = int(sys.argv[3]) if len(sys.argv) > 3 else 40
keys = workload.generate_keys(bht.mix_seed(1, 0x6B657973), n, device=0).keys.view(torch.int32)
vals = bht.values_for_keys(keys)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
CONFIGS = [("0", "", "")] + [("1", lf_, d_) for lf_ in ("0.96", "0.975", "0.985") for d_ in ("24", "4")] + [("1", "0.98", "12"), ("1", "0.98", "1")]
if len(sys.argv) > 4:
    CONFIGS = [tuple(c.split(":")) for c in sys.argv[4:]]
for thr, tail_lf, div in CONFIGS:
    os.environ["BHT_TAIL_THROTTLE"] = thr; bht.reload_tuning()
    if tail_lf:
        os.environ["BHT_TAIL_LF"], os.environ["BHT_TAIL_DIV"] = tail_lf, div; bht.reload_tuning()
    ok, dropped, ms = 0, 0, 0.0
    for t in range(trials):
        cfg = bht.make_config("bcht", n, lf, 16, seed=bht.mix_seed(1234, t))
        table = bht.HashTable(cfg, 0)
        ev0.record(); table.insert(keys, vals, want_result=False); ev1.record(); ev1.synchronize()
        ms += ev0.elapsed_time(ev1)
        o = table.last_insert_result()
        ok += o.success
        dropped += o.failed
        table.close()
    rate = ok / trials
    print(f"throttle={thr} tail_lf={tail_lf or '-':>5s} div={div or '-':>3s}: {ok}/{trials} builds succeed, {dropped} dropped, {ms / trials:.3f} ms per build, "
          f"{ms / trials / max(rate, 1e-9):.2f} ms per successful build", flush=True)
