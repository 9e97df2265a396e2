"""One setup, truncated schedule — short kernel for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl
which = sys.argv[1] if len(sys.argv) > 1 else "C1"
nset = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = wl.config(which)
inp = wl.build_inputs(cfg, limit=nset)
s = wl.scores_for(cfg)
eng = rw.Engine(0)
eng.load_scores(s)
eng.load_profiles(inp.koff, inp.kx, inp.ky)
tau = cfg.taus[0]
opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
for _ in range(2):
    recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
ms = eng.last_kernel_ms()
p = int(recs["eval_passes"].sum()); pp = int(recs["polish_passes"].sum())
print(f"kernel {ms:.3f} ms, eval passes {p}, polish passes {pp}, us/pass {ms*1e3/p*len(recs):.2f}")
eng.set_profiling(True)
recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
pr = eng.profile()
tot = eng.last_kernel_ms() * 1.965e6
print("cycles: phase1 %.0f phase2 %.0f walk %.0f polish %.0f polish_misses %d  (kernel ~%.0f cyc)" % (pr[0], pr[1], pr[2], pr[3], pr[4], tot))
print("per eval pass: p1 %.0f p2 %.0f walk %.0f" % (pr[0]/p, pr[1]/p, pr[2]/p))
