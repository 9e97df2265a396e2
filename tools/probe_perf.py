"""Quick perf probe: C1 sweep at full default schedule on one GPU."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl

which = sys.argv[1] if len(sys.argv) > 1 else "C1"
limit = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = wl.config(which)
inp = wl.build_inputs(cfg, limit=limit)
s = wl.scores_for(cfg)
eng = rw.Engine(0)
eng.load_scores(s)
eng.load_profiles(inp.koff, inp.kx, inp.ky)
tau = cfg.taus[0]
opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
bp = rw.BetaSearchParams()
if len(sys.argv) > 3 and sys.argv[3] == "trunc":
    bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
t = time.time()
recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
wall = time.time() - t
ms = eng.last_kernel_ms()
passes = int(recs["eval_passes"].sum())
print(f"{which}: setups={len(recs)} wall={wall:.3f}s kernel={ms:.1f}ms passes={passes} "
      f"passes/setup={passes/len(recs):.0f} evals/s={passes*cfg.n/(ms/1e3):.3e} "
      f"us/pass/setup={ms*1e3/ (passes/len(recs)):.2f}")
best = rw.reduce_records(recs)
print("winner", best, recs[best]["setup_id"] if best >= 0 else None, recs[best]["score"] if best>=0 else None,
      "feasible", int(recs["feasible"].sum()))
