"""Synthetic workloads of BASELINE.json's configs, built from the host
input producers (rw_synth_scores, rw_enumerate_retain) — no oracle involved.

Profile formula: model i at (tp, rho) has knots
    (0, b), (20, b + 20 s), (60, b + 140 s),  b = (20 + 25 i) / (sqrt(tp) rho),
    s = (1 + 1.5 i) / (tp rho);  memory m(tp=1) = 0.4, m(tp=2) = 0.25.
C4 uses 12-knot nonlinear curves b + s L + c / (1 - L / L_max) up to 0.95 L_max.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import routeplan as rp


def beta_shapes(m: int) -> List[Tuple[float, float]]:
    """Evenly spaced from (2, 8) to (8, 2) across models."""
    if m == 1:
        return [(5.0, 5.0)]
    return [(2.0 + 6.0 * i / (m - 1), 8.0 - 6.0 * i / (m - 1)) for i in range(m)]


def linear_knots(i: int, tp: int, rho: float):
    b = (20.0 + 25.0 * i) / (math.sqrt(tp) * rho)
    s = (1.0 + 1.5 * i) / (tp * rho)
    return [(0.0, b), (20.0, b + 20.0 * s), (60.0, b + 140.0 * s)]


def nonlinear_knots(i: int, tp: int, rho: float, k: int = 12):
    b = (20.0 + 10.0 * (i % 8)) / (math.sqrt(tp) * rho)
    s = (0.5 + 0.25 * (i % 5)) / (tp * rho)
    c = 5.0 + i
    lmax = 30.0 * tp * rho
    xs = [0.95 * lmax * q / (k - 1) for q in range(k)]
    return [(x, b + s * x + c / (1.0 - x / lmax)) for x in xs]


@dataclass
class SweepConfig:
    name: str
    n: int
    models: List[str]
    tp_choices: List[List[int]]
    rho_choices: List[List[float]]
    gpu_count: int
    rho_floor: float
    lambda_rps: float
    taus: List[float]
    kappa: float = 1.25
    nonlinear: bool = False
    ties: bool = False
    seed: int = 1
    mem: dict = field(default_factory=dict)

    @property
    def m(self):
        return len(self.models)


def config(name: str, n: Optional[int] = None) -> SweepConfig:
    """BASELINE.json configs C1..C5 (n may be overridden for parity-sized runs)."""
    if name == "C1":
        c = SweepConfig("C1: 10k x 4 x 64, single SLO", 10_000, list("ABCD"),
                        [[1, 2], [1, 2], [1], [1]], [[0.5, 1.0]] * 4, 8, 0.1, 40.0, [120.0])
    elif name == "C2":
        rhos = [0.25, 0.5, 0.75, 1.0]
        c = SweepConfig("C2: 100k x 4 x 512, 8 SLOs", 100_000, list("ABCD"),
                        [[1, 2], [1, 2], [1, 2], [1]], [rhos, rhos, rhos, [1.0]], 8, 0.1, 40.0,
                        [60.0, 80.0, 100.0, 120.0, 140.0, 160.0, 200.0, 250.0])
    elif name == "C3":
        c = SweepConfig("C3: 1M x 8 x 4096 incl. TP", 1_000_000, list("ABCDEFGH"),
                        [[1, 2]] * 8, [[0.5, 1.0]] * 4 + [[1.0]] * 4, 16, 0.1, 80.0, [100.0])
    elif name == "C4":
        models = [f"M{i:02d}" for i in range(16)]
        c = SweepConfig("C4: 10M x 16 x 16384, nonlinear", 10_000_000, models,
                        [[1, 2]] * 14 + [[1]] * 2, [[1.0]] * 16, 32, 0.1, 160.0, [150.0],
                        nonlinear=True)
    elif name == "C5":
        c = SweepConfig("C5: 1M x 8 x 1024, adversarial ties", 1_000_000, list("ABCDEFGH"),
                        [[1, 2]] * 5 + [[1]] * 3, [[0.5, 1.0]] * 5 + [[1.0]] * 3, 16, 0.1, 80.0,
                        [100.0], ties=True)
    else:
        raise KeyError(name)
    if n is not None:
        c.n = n
    c.mem = {(mdl, tp): (0.4 if tp == 1 else 0.25) for mdl in c.models for tp in (1, 2)}
    return c


def scores_for(cfg: SweepConfig, synth=None) -> np.ndarray:
    """synth(n, shapes, seed) -> matrix overrides the host producer (the bench's reference
    arm passes the reference library's own synth_scores, so it loads nothing of ours)."""
    if synth is None:
        s = rp.synth_scores(cfg.n, cfg.models, beta_shapes(cfg.m), cfg.seed).scores
    else:
        s = synth(cfg.n, beta_shapes(cfg.m), cfg.seed)
    if cfg.ties:
        s = tie_scores(s, cfg.seed)
    return s


def tie_scores(s: np.ndarray, seed: int) -> np.ndarray:
    """C5: quantise to k/16; 10% of rows get a duplicated column or a 1-ulp neighbour."""
    q = np.round(s * 16.0) / 16.0
    rng = np.random.default_rng(seed)
    n, m = q.shape
    rows = rng.choice(n, size=max(1, n // 10), replace=False)
    for j in rows:
        a, b = rng.choice(m, size=2, replace=False)
        if rng.random() < 0.5:
            q[j, b] = q[j, a]
        else:
            v = q[j, a]
            q[j, b] = np.nextafter(v, 1.0) if v < 1.0 else np.nextafter(v, 0.0)
    return np.clip(q, 0.0, 1.0)


@dataclass
class SweepInputs:
    cfg: SweepConfig
    space: rp.SetupSpace
    mem: rp.MemoryTable
    lib: rp.ProfileLibrary
    retained: np.ndarray          # enumeration ids of retained setups
    tp: np.ndarray                # [retained, M]
    rho: np.ndarray               # [retained, M]
    profile_keys: List[tuple]     # (model index, tp, rho) per table row
    koff: np.ndarray
    kx: np.ndarray
    ky: np.ndarray
    profile_index: np.ndarray     # [retained, M] int32
    enumerated: int


class _SpaceView:
    """The plain setup-space description an external enumerate/retain takes."""

    def __init__(self, cfg: SweepConfig):
        self.tp_choices = [list(t) for t in cfg.tp_choices]
        self.rho_choices = [list(r) for r in cfg.rho_choices]
        self.memory = [(cfg.models.index(mdl), tp, f) for (mdl, tp), f in cfg.mem.items()]
        self.gpu_count, self.rho_floor = cfg.gpu_count, cfg.rho_floor


def build_inputs(cfg: SweepConfig, limit: Optional[int] = None,
                 enumerate_fn=None) -> SweepInputs:
    """enumerate_fn(space_view) -> (verdict, tp, rho) overrides the host enumerate/retain
    (the bench's reference arm passes the reference library's own)."""
    space = rp.SetupSpace(list(cfg.models), [list(t) for t in cfg.tp_choices],
                          [list(r) for r in cfg.rho_choices])
    mem = rp.MemoryTable()
    for (mdl, tp), f in cfg.mem.items():
        mem.insert(mdl, tp, f)
    if enumerate_fn is None:
        verdict, tps, rhos = rp.enumerate_retain(space, cfg.gpu_count, cfg.rho_floor, mem)
    else:
        verdict, tps, rhos = enumerate_fn(_SpaceView(cfg))
    retained = np.nonzero(verdict == 0)[0]
    if limit is not None:
        retained = retained[:limit]
    lib = rp.ProfileLibrary()
    keys, index = [], {}
    koff, kx, ky = [0], [], []
    pidx = np.zeros((len(retained), cfg.m), np.int32)
    for i, mdl in enumerate(cfg.models):
        for tp in cfg.tp_choices[i]:
            for rho in cfg.rho_choices[i]:
                knots = nonlinear_knots(i, tp, rho) if cfg.nonlinear else linear_knots(i, tp, rho)
                lib.add(rp.LatencyProfile(mdl, tp, rho, rp.Metric.TTFT, knots))
                index[(i, tp, rp.quantize_rho(rho))] = len(keys)
                keys.append((i, tp, rho))
                for x, y in knots:
                    kx.append(x)
                    ky.append(y)
                koff.append(len(kx))
    for r, k in enumerate(retained):
        for i in range(cfg.m):
            pidx[r, i] = index[(i, int(tps[k, i]), rp.quantize_rho(float(rhos[k, i])))]
    return SweepInputs(cfg, space, mem, lib, retained.astype(np.int64), tps[retained],
                       rhos[retained], keys, np.array(koff, np.int64), np.array(kx, np.float64),
                       np.array(ky, np.float64), pidx, len(verdict))


def truncated_params(span_div: float = 4.0) -> rp.BetaSearchParams:
    """BASELINE.md's truncated schedule for C2-C5 parity / CPU timing:
    subgradient max_iters=20, PGA max_iters=5, beta epsilon = span/4."""
    return rp.BetaSearchParams(beta_min=0.0, beta_max=-1.0, epsilon=-1.0,
                               pga=rp.PgaParams(eta=0.05, max_iters=5, w_tol=1e-10,
                                                dual=rp.SubgradientParams(1.0, 20, 1e-12, 4)))


def with_span_epsilon(p: rp.BetaSearchParams, tau: float, div: float) -> rp.BetaSearchParams:
    hi = p.beta_max if p.beta_max >= 0 else 10.0 / tau
    return rp.BetaSearchParams(p.beta_min, p.beta_max, (hi - p.beta_min) / div, p.pga)
