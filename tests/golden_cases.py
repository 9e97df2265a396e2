"""Loader for tests/golden/reference_cases.json (written by oracle/golden_gen.cpp from the
UNMODIFIED reference library on the reference's own doctest instances).  Hex-float
strings decode to the exact doubles the reference produced."""
from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "reference_cases.json")


def _f(x):
    return float.fromhex(x) if isinstance(x, str) else float(x)


def _fv(v):
    return np.array([_f(x) for x in v], np.float64)


def _dec(k, v):
    if isinstance(v, dict):
        return {kk: _dec(kk, vv) for kk, vv in v.items()}
    if isinstance(v, str):
        return _f(v)
    if isinstance(v, list):
        if v and isinstance(v[0], str):
            return _fv(v)
        return np.array(v, np.int64) if v else np.zeros(0)
    return v


@functools.lru_cache(maxsize=1)
def load():
    with open(GOLDEN) as f:
        raw = json.load(f)
    mats = [_fv(m["v"]).reshape(m["n"], m["m"]) for m in raw["matrices"]]
    cases = []
    for c in raw["cases"]:
        d = {}
        for k, v in c.items():
            if k == "scores":
                d[k] = mats[v]
            elif k in ("kind", "cite"):
                d[k] = v
            elif k == "profiles":
                d[k] = [[(_f(a), _f(b)) for a, b in p] for p in v]
            else:
                d[k] = _dec(k, v)
        cases.append(d)
    return cases


def of_kind(kind):
    return [c for c in load() if c["kind"] == kind]


def ids(cases):
    return [f"{i}:{c['cite']}" for i, c in enumerate(cases)]


def params_from(case):
    """oracle.Params for a solve / optfrac / optbeta case."""
    from oracle import Params
    p = case["params"]
    if case["kind"] == "solve":
        return Params(eta0=p["eta0"], sub_max_iters=p["max_iters"],
                      residual_tol=p["residual_tol"], polish_passes=p["polish_passes"])
    pga = p if case["kind"] == "optfrac" else p["pga"]
    d = pga["dual"]
    kw = dict(eta0=d["eta0"], sub_max_iters=d["max_iters"], residual_tol=d["residual_tol"],
              polish_passes=d["polish_passes"], pga_eta=pga["eta"],
              pga_max_iters=pga["max_iters"], w_tol=pga["w_tol"])
    if case["kind"] == "optbeta":
        kw.update(beta_min=p["beta_min"], beta_max=p["beta_max"], epsilon=p["epsilon"])
    return Params(**kw)


def bits(x):
    return np.asarray(x, np.float64).view(np.int64)
