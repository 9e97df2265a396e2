"""GPU parity against the reference's own outputs: every case of
tests/golden/reference_cases.json (the reference's doctest instances run through the
UNMODIFIED reference library, oracle/golden_gen.cpp) replayed through the C-ABI on the
sm_100a kernels.  Bar: bit-exact."""
import numpy as np
import pytest

import golden_cases as G
import paper_2604_10907_b200 as rw
from golden_cases import bits

pytestmark = pytest.mark.gpu

EVAL = G.of_kind("eval")
SOLVE = G.of_kind("solve")
SIMPLEX = G.of_kind("simplex")
LATENCY = G.of_kind("latency")
OPTFRAC = G.of_kind("optfrac")
OPTBETA = G.of_kind("optbeta")


def _knots(profiles):
    koff, kx, ky = [0], [], []
    for p in profiles:
        for x, y in p:
            kx.append(x)
            ky.append(y)
        koff.append(len(kx))
    return np.array(koff, np.int64), np.array(kx), np.array(ky)


def _sub(p):
    return rw.SubgradientParams(p["eta0"], int(p["max_iters"]), p["residual_tol"],
                                int(p["polish_passes"]))


def _pga(p):
    return rw.PgaParams(p["eta"], int(p["max_iters"]), p["w_tol"], _sub(p["dual"]))


@pytest.mark.parametrize("case", EVAL, ids=G.ids(EVAL))
def test_eval_golden(eng, case):
    eng.load_scores(case["scores"])
    g = eng.dual_objective(case["c"], case["alpha"])
    mo, counts = eng.assign_prompts(case["alpha"])
    assert bits(g) == bits(case["g"])
    assert counts.tolist() == case["counts"].tolist()
    assert mo.tolist() == case["model_of"].tolist()


@pytest.mark.parametrize("case", SOLVE, ids=G.ids(SOLVE))
def test_solve_golden(eng, case):
    eng.load_scores(case["scores"])
    init = case["init_alpha"] if len(case["init_alpha"]) else None
    got = eng.solve_dual(case["c"], _sub(case["params"]), init)
    assert np.array_equal(bits(got.alpha_star.alpha), bits(case["alpha_star"]))
    assert bits(got.score) == bits(case["score"])
    assert bits(got.dual_bound) == bits(case["dual_bound"])
    assert bits(got.duality_gap) == bits(case["duality_gap"])
    assert got.assignment == case["assignment"].tolist()
    assert np.array_equal(bits(got.count_residual), bits(case["count_residual"]))
    assert got.iterations == case["iterations"] and got.converged == bool(case["converged"])


@pytest.mark.parametrize("case", SIMPLEX, ids=G.ids(SIMPLEX))
def test_simplex_golden(eng, case):
    assert np.array_equal(bits(eng.project_simplex(case["v"])), bits(case["w"]))


@pytest.mark.parametrize("case", LATENCY, ids=G.ids(LATENCY))
def test_latency_golden(eng, case):
    m = len(case["w"])
    eng.load_scores(np.zeros((1, m)))
    eng.load_profiles(*_knots(case["profiles"]))
    r = eng.system_latency_eval(np.arange(m), case["w"], case["lambda"], case["kappa"])
    assert bits(r["latency"]) == bits(case["latency"])
    assert np.array_equal(bits(r["loads"]), bits(case["loads"]))
    assert np.array_equal(bits(r["lats"]), bits(case["lats"]))
    assert r["oor"].tolist() == case["oor"].tolist()
    assert np.array_equal(bits(r["grad"]), bits(case["grad"]))


@pytest.mark.parametrize("case", OPTFRAC, ids=G.ids(OPTFRAC))
def test_optfrac_golden(eng, case):
    m = case["scores"].shape[1]
    eng.load_scores(case["scores"])
    eng.load_profiles(*_knots(case["profiles"]))
    ctx = case["ctx"]
    opt = rw.OptimizeContext(lambda_rps=ctx["lambda_rps"], tau_ms=ctx["tau_ms"],
                             kappa=ctx["kappa"])
    got = eng.optimize_fractions(np.arange(m), case["beta"], opt, _pga(case["params"]))
    assert np.array_equal(bits(got.w.w), bits(case["w"]))
    assert bits(got.objective) == bits(case["objective"])
    assert bits(got.score) == bits(case["score"])
    assert bits(got.latency_ms) == bits(case["latency_ms"])
    assert got.iterations == case["iterations"] and got.converged == bool(case["converged"])
    assert got.out_of_range == [bool(x) for x in case["out_of_range"]]


@pytest.mark.parametrize("case", OPTBETA, ids=G.ids(OPTBETA))
def test_optbeta_golden(eng, case):
    m = case["scores"].shape[1]
    eng.load_scores(case["scores"])
    eng.load_profiles(*_knots(case["profiles"]))
    ctx = case["ctx"]
    p = case["params"]
    opt = rw.OptimizeContext(lambda_rps=ctx["lambda_rps"], tau_ms=ctx["tau_ms"],
                             kappa=ctx["kappa"])
    bp = rw.BetaSearchParams(p["beta_min"], p["beta_max"], p["epsilon"], _pga(p["pga"]))
    got = eng.optimize_beta(np.arange(m), opt, bp)
    assert got.feasible == bool(case["feasible"])
    assert (got.beta_star is not None) == bool(case["has_beta_star"])
    assert len(got.trace) == len(case["trace_beta"])
    for st, b, sc, lt, ok in zip(got.trace, case["trace_beta"], case["trace_score"],
                                 case["trace_latency"], case["trace_ok"]):
        assert bits(st.beta) == bits(b) and bits(st.score) == bits(sc)
        assert bits(st.latency_ms) == bits(lt) and st.feasible == bool(ok)
    if got.feasible:
        b = case["best"]
        assert bits(got.beta_star) == bits(case["beta_star"])
        assert np.array_equal(bits(got.w_star.w), bits(case["w_star"]))
        assert np.array_equal(bits(got.best.w.w), bits(b["w"]))
        assert bits(got.best.score) == bits(b["score"])
        assert bits(got.best.latency_ms) == bits(b["latency_ms"])
        assert bits(got.best.objective) == bits(b["objective"])
