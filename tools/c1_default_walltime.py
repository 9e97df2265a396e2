#!/usr/bin/env python3
"""Wall time to the optimal setup, C1 at the reference defaults (config.hpp:20-31):
10k prompts x 4 models x 64 retained setups, tau = 120 ms — the configuration the survey
timed on the reference CPU solver (404.5 s on 8 threads).  64 setups fill 64 of the
B200's 296 CTA slots, so the sweep is latency-bound: the speculative bisection (f4,
rw_sweep_spec) evaluates 2-3 levels of every setup's beta bisection per launch.
Prints one JSON line per variant (records must be bit-identical to the sequential sweep)
and, with --ref, times the reference select_setup on this host's cores.
Usage: python tools/c1_default_walltime.py [--ref]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2604_10907_b200 as rw  # noqa: E402
from paper_2604_10907_b200 import workloads as wl  # noqa: E402


def main():
    cfg = wl.config("C1")
    inp = wl.build_inputs(cfg)
    s = wl.scores_for(cfg)
    eng = rw.Engine(0)
    eng.load_scores(s)
    eng.load_profiles(inp.koff, inp.kx, inp.ky)
    tau = cfg.taus[0]
    p = rw.BetaSearchParams()  # reference defaults
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
    base = None
    for name, fn in [("sequential (rw_sweep)", lambda: eng.sweep(inp.profile_index, inp.retained, opt, p)),
                     ("speculative depth 2 (rw_sweep_spec)",
                      lambda: eng.sweep_spec(inp.profile_index, inp.retained, [tau], opt, p, 2)),
                     ("speculative depth 3 (rw_sweep_spec)",
                      lambda: eng.sweep_spec(inp.profile_index, inp.retained, [tau], opt, p, 3))]:
        t0 = time.perf_counter()
        recs = fn()
        dt = time.perf_counter() - t0
        win = rw.reduce_records(recs)
        same = None
        if base is None:
            base = recs
        else:
            same = all(np.ascontiguousarray(base[f]).tobytes() == np.ascontiguousarray(recs[f]).tobytes()
                       for f in base.dtype.names if f != "exec_passes")
        print(json.dumps({"variant": name, "wall_s": dt, "setups": len(recs),
                          "winner_setup": int(recs[win]["setup_id"]) if win >= 0 else None,
                          "winner_score": float(recs[win]["score"]) if win >= 0 else None,
                          "reference_passes": int(recs["eval_passes"].sum()),
                          "executed_passes": int(recs["exec_passes"].sum()),
                          "records_identical_to_sequential": same}), flush=True)
    if "--ref" in sys.argv:
        from oracle import Params, ProfileTable, Reference
        R = Reference()

        class Sp:
            pass
        sp = Sp()
        sp.tp_choices = [list(t) for t in cfg.tp_choices]
        sp.rho_choices = [list(r) for r in cfg.rho_choices]
        sp.memory = [(cfg.models.index(mdl), tp, f) for (mdl, tp), f in cfg.mem.items()]
        sp.profile_keys = inp.profile_keys
        sp.profiles = ProfileTable(inp.koff, inp.kx, inp.ky)
        sp.gpu_count, sp.rho_floor = cfg.gpu_count, cfg.rho_floor
        sp.lambda_rps, sp.tau_ms, sp.kappa = cfg.lambda_rps, tau, cfg.kappa
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        out = R.select_setup(s, sp, Params(), parallelism=threads)
        dt = time.perf_counter() - t0
        same = np.array_equal(out["sweep_score"].view(np.int64), base["score"].view(np.int64))
        print(json.dumps({"variant": f"reference select_setup ({threads} threads)", "wall_s": dt,
                          "winner_score": float(out["score"]),
                          "records_identical_to_gpu": bool(same)}), flush=True)


if __name__ == "__main__":
    main()
