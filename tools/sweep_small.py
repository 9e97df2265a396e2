"""One small truncated-schedule sweep (debug helper: run under compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
limit = int(sys.argv[3]) if len(sys.argv) > 3 else 6
cfg = wl.config(name, n=n)
inp = wl.build_inputs(cfg, limit=limit)
s = wl.scores_for(cfg)
eng = rw.Engine(0)
eng.load_scores(s)
eng.load_profiles(inp.koff, inp.kx, inp.ky)
tau = cfg.taus[0]
bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
print(name, n, limit, "ok", [float(r["score"]) for r in recs])
