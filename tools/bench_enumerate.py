#!/usr/bin/env python3
"""f1 timing: setup enumeration + retention at 1e5-1e6 candidates — the
host step that directly precedes the sweep.  Ours: rw_enumerate_retain (host C++, threads
over the enumeration range).  Reference: enumerate_setups + retain through oracle/_ref
(setup_search.cpp:99-152, std::set FFD, one thread).  Verdicts must agree exactly.
Usage: python tools/bench_enumerate.py   (CPU only; prints one line per space)"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2604_10907_b200 import workloads as wl  # noqa: E402
from paper_2604_10907_b200 import routeplan as rp  # noqa: E402
from oracle import Reference  # noqa: E402


def space(n_models, tps, rhos, gpus):
    cfg = wl.config("C3")
    cfg.models = [f"M{i:02d}" for i in range(n_models)]
    cfg.tp_choices = [list(tps)] * n_models
    cfg.rho_choices = [list(rhos)] * n_models
    cfg.gpu_count = gpus
    cfg.mem = {(mdl, tp): (0.4 if tp == 1 else (0.25 if tp == 2 else 0.15))
               for mdl in cfg.models for tp in (1, 2, 4)}
    return cfg


def main():
    R = Reference()
    cases = [("C3 space: 8 models (4096 candidates) on 16 GPUs", space(8, [1, 2], [0.5, 1.0], 16)),
             ("9 models x (tp{1,2} x rho{.5,1}) on 16 GPUs (2.6e5)", space(9, [1, 2], [0.5, 1.0], 16)),
             ("10 models x (tp{1,2} x rho{.5,1}) on 16 GPUs (1.0e6)",
              space(10, [1, 2], [0.5, 1.0], 16)),
             ("12 models x (tp{1,2} x rho{.5,1}) on 24 GPUs (1.7e7)",
              space(12, [1, 2], [0.5, 1.0], 24))]
    for label, cfg in cases:
        sp = wl._SpaceView(cfg)
        s = rp.SetupSpace(list(cfg.models), sp.tp_choices, sp.rho_choices)
        mem = rp.MemoryTable()
        for (mdl, tp), f in cfg.mem.items():
            mem.insert(mdl, tp, f)
        t0 = time.perf_counter()
        v_ours, _, _ = rp.enumerate_retain(s, cfg.gpu_count, cfg.rho_floor, mem)
        t_enum = time.perf_counter() - t0
        t0 = time.perf_counter()
        v_ref, _, _ = R.enumerate_retain(sp)
        t_ref = time.perf_counter() - t0
        same = np.array_equal(v_ours, v_ref[: len(v_ours)])
        print(f"{label}: {len(v_ours)} candidates, {int((v_ours == 0).sum())} retained; "
              f"ours {t_enum * 1e3:.1f} ms ({os.cpu_count()} host threads), reference "
              f"{t_ref * 1e3:.1f} ms (1 thread), x{t_ref / t_enum:.1f}; verdicts identical: "
              f"{same}",
              flush=True)


if __name__ == "__main__":
    main()
