"""One sweep on a truncated schedule with the diagnostics counters (rw_get_profile)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl
which = sys.argv[1] if len(sys.argv) > 1 else "C2"
nset = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sched = sys.argv[3] if len(sys.argv) > 3 else "trunc"
n_over = int(sys.argv[4]) if len(sys.argv) > 4 else None
cfg = wl.config(which, n_over)
inp = wl.build_inputs(cfg, limit=nset)
s = wl.scores_for(cfg)
eng = rw.Engine(0)
eng.load_scores(s)
eng.load_profiles(inp.koff, inp.kx, inp.ky)
tau = cfg.taus[0]
opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0) if sched == "trunc" else rw.BetaSearchParams()
recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
eng.set_profiling(True)
recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
ms = eng.last_kernel_ms()
pr = eng.profile()
p = int(recs["exec_passes"].sum()); pp = int(recs["polish_passes"].sum())
pref = int(recs["eval_passes"].sum())
ctas = min(len(recs), 296)
cyc = ms * 1.965e6
names = ["load(w0)", "totbar(w0)", "empty(w0)", "polish", "pmiss", "pradix", "walk_wait",
         "walk_busy", "fast_blocks", "slow_blocks", "raw_rows", "psweep", "pselect", "pass",
         "repair", "p1_rounds", "p2_passes", "moves", "p_over", "p_far", "p_shell", "p_move", "p2_refresh", "p1_cyc", "p2_cyc", "ref_cyc", "p2_seed", "p_hist", "-", "p2_merge", "p_fhit", "p_fused"]
print(f"{which} x{len(recs)} ({sched}): kernel {ms:.3f} ms (~{cyc:.3e} cyc/CTA), eval passes {p}, "
      f"(reference trajectory {pref}), polish passes {pp}, evals/s {p * cfg.n / (ms / 1e3):.3e}")
for i, nm in enumerate(names):
    v = pr[i]
    if nm in ("pmiss", "pradix", "fast_blocks", "slow_blocks", "raw_rows", "p1_rounds", "p2_passes", "moves", "p_over", "p_far", "p_shell", "p2_refresh", "p_hist", "p2_merge", "p_fhit"):
        print(f"  {nm:12s} {v:14d}  per pass {v / max(p, 1):10.2f}")
    elif nm == "p_move":
        ncoord = max(pp * cfg.m, 1)
        print(f"  {nm:12s} mean log2(|move|/d) over nonzero moves ~ {v / ncoord - 64:8.2f} (all coords {ncoord})")
    elif nm != "-":
        print(f"  {nm:12s} {v / ctas:14.3e} cyc/CTA  {100.0 * v / ctas / cyc:5.1f}%  per pass {v / max(p, 1):10.0f}")
