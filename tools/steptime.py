import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl
cfg = wl.config("C2"); inp = wl.build_inputs(cfg); s = wl.scores_for(cfg)
taus = np.array(cfg.taus)
dev = torch.device("cuda", 0)
eng = rw.Engine(0); st = torch.cuda.current_stream(dev); eng.set_stream(st.cuda_stream)
sd = torch.from_numpy(s).to(dev); eng.bind_scores_device(sd.data_ptr(), cfg.n, cfg.m)
eng.load_profiles(inp.koff, inp.kx, inp.ky)
opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=float(taus[0]), kappa=cfg.kappa)
pg = [wl.with_span_epsilon(wl.truncated_params(), float(t), 4.0) for t in taus]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for it in range(4):
    t0 = time.perf_counter(); flush.fill_(1); torch.cuda.synchronize(); t1 = time.perf_counter()
    eng.sweep_async(inp.profile_index, inp.retained, opt, pg, 0, 1, taus=taus); t2 = time.perf_counter()
    r = eng.sweep_fetch(); t3 = time.perf_counter()
    print(f"fill {1e3*(t1-t0):.1f} ms, async {1e3*(t2-t1):.1f} ms, fetch {1e3*(t3-t2):.1f} ms, kernel {eng.last_kernel_ms():.1f} ms")
