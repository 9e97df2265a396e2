"""Per-pass cost probe: K eval passes at fixed prices on one CTA."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl
from paper_2604_10907_b200._abi import dptr
which = sys.argv[1] if len(sys.argv) > 1 else "C1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = wl.config(which)
s = wl.scores_for(cfg)
eng = rw.Engine(0)
eng.load_scores(s)
m = cfg.m
c = np.full(m, cfg.n / m)
alpha = np.linspace(0.0, 0.3, m)
g = C.c_double()
eng.set_profiling(True)
for rep in range(2):
    eng._chk(eng.L.rw_bench_passes(eng.h, dptr(c), dptr(alpha), K, C.byref(g)))
    ms = eng.last_kernel_ms()
    pr = eng.profile()
print(f"{which}: {K} passes in {ms:.3f} ms -> {ms*1e3/K:.2f} us/pass, {cfg.n*K/(ms/1e3):.3e} evals/s (1 CTA)")
print("per pass cycles: p1 %.0f p2 %.0f walk %.0f" % (pr[0]/K, pr[1]/K, pr[2]/K))
