"""Pins the checker (CPU, no GPU).

1. The plain-C restatement (oracle/rw_oracle.c) reproduces, bit for bit, what the
   UNMODIFIED reference library returned on the reference's own doctest instances
   (tests/golden/reference_cases.json, made by oracle/golden_gen.cpp).
2. Where oracle/_ref (the reference compiled from /root/reference sources) is present,
   the restatement also matches it live on larger seeded instances, down to the
   per-setup records of select_setup.
3. The worked examples of the reference tests hold for the restatement directly.
"""
import numpy as np
import pytest

import golden_cases as G
from golden_cases import bits

EVAL = G.of_kind("eval")
SOLVE = G.of_kind("solve")
SIMPLEX = G.of_kind("simplex")
LATENCY = G.of_kind("latency")
OPTFRAC = G.of_kind("optfrac")
OPTBETA = G.of_kind("optbeta")


def test_fixture_covers_every_kind():
    assert len(EVAL) > 200 and len(SOLVE) > 100 and len(SIMPLEX) > 100
    assert len(LATENCY) > 40 and len(OPTFRAC) >= 5 and len(OPTBETA) >= 8


@pytest.mark.parametrize("case", EVAL, ids=G.ids(EVAL))
def test_eval_dual_golden(oracle, case):
    g, counts, mo = oracle.eval_dual(case["scores"], case["c"], case["alpha"])
    assert bits(g) == bits(case["g"])
    assert counts.tolist() == case["counts"].tolist()
    assert mo.tolist() == case["model_of"].tolist()


@pytest.mark.parametrize("case", SOLVE, ids=G.ids(SOLVE))
def test_solve_dual_golden(oracle, case):
    init = case["init_alpha"] if len(case["init_alpha"]) else None
    r = oracle.solve_dual(case["scores"], case["c"], G.params_from(case), init_alpha=init)
    assert np.array_equal(bits(r["alpha"]), bits(case["alpha_star"]))
    assert bits(r["score"]) == bits(case["score"])
    assert bits(r["dual_bound"]) == bits(case["dual_bound"])
    assert bits(r["gap"]) == bits(case["duality_gap"])
    assert r["assignment"].tolist() == case["assignment"].tolist()
    assert np.array_equal(bits(r["residual"]), bits(case["count_residual"]))
    assert r["iterations"] == case["iterations"] and r["converged"] == bool(case["converged"])
    if "exact" in case:  # strong duality (test_score_dual.cpp:151-164)
        assert abs(r["score"] - case["exact"]) <= 1e-6


@pytest.mark.parametrize("case", SIMPLEX, ids=G.ids(SIMPLEX))
def test_project_simplex_golden(oracle, case):
    assert np.array_equal(bits(oracle.project_simplex(case["v"])), bits(case["w"]))


def _table(profiles):
    from oracle import ProfileTable
    return ProfileTable.from_lists(profiles)


@pytest.mark.parametrize("case", LATENCY, ids=G.ids(LATENCY))
def test_latency_golden(oracle, case):
    m = len(case["w"])
    r = oracle.latency_eval(_table(case["profiles"]), np.arange(m), case["w"], case["lambda"],
                            case["kappa"])
    assert bits(r["latency"]) == bits(case["latency"])
    assert np.array_equal(bits(r["loads"]), bits(case["loads"]))
    assert np.array_equal(bits(r["lats"]), bits(case["lats"]))
    assert r["oor"].tolist() == case["oor"].tolist()
    assert np.array_equal(bits(r["grad"]), bits(case["grad"]))


@pytest.mark.parametrize("case", OPTFRAC, ids=G.ids(OPTFRAC))
def test_optimize_fractions_golden(oracle, case):
    m = case["scores"].shape[1]
    ctx = case["ctx"]
    r = oracle.optimize_fractions(case["scores"], _table(case["profiles"]), np.arange(m),
                                  case["beta"], ctx["lambda_rps"], ctx["tau_ms"], ctx["kappa"],
                                  G.params_from(case))
    assert np.array_equal(bits(r["w"]), bits(case["w"]))
    assert bits(r["objective"]) == bits(case["objective"])
    assert bits(r["score"]) == bits(case["score"])
    assert bits(r["latency_ms"]) == bits(case["latency_ms"])
    assert r["iterations"] == case["iterations"] and r["converged"] == bool(case["converged"])
    assert r["oor"].tolist() == case["out_of_range"].tolist()


@pytest.mark.parametrize("case", OPTBETA, ids=G.ids(OPTBETA))
def test_optimize_beta_golden(oracle, case):
    m = case["scores"].shape[1]
    ctx = case["ctx"]
    r = oracle.optimize_beta(case["scores"], _table(case["profiles"]), np.arange(m),
                             ctx["lambda_rps"], ctx["tau_ms"], ctx["kappa"], G.params_from(case))
    assert r["feasible"] == bool(case["feasible"])
    assert r["has_beta_star"] == bool(case["has_beta_star"])
    assert bits(r["beta_star"]) == bits(case["beta_star"])
    assert r["n_trace"] == len(case["trace_beta"])
    assert np.array_equal(bits(r["trace_beta"]), bits(case["trace_beta"]))
    assert np.array_equal(bits(r["trace_score"]), bits(case["trace_score"]))
    assert np.array_equal(bits(r["trace_latency"]), bits(case["trace_latency"]))
    assert r["trace_ok"].tolist() == case["trace_ok"].tolist()
    if r["feasible"]:
        b = case["best"]
        assert np.array_equal(bits(r["w_star"]), bits(case["w_star"]))
        assert np.array_equal(bits(r["best_w"]), bits(b["w"]))
        assert bits(r["best_score"]) == bits(b["score"])
        assert bits(r["best_latency"]) == bits(b["latency_ms"])
        assert bits(r["best_objective"]) == bits(b["objective"])


# ---- worked examples straight from the reference tests -------------------------------

def test_worked_examples(oracle):
    s = np.array([[0.9, 0.8], [0.4, 0.7]])
    g, counts, mo = oracle.eval_dual(s, np.array([1.0, 1.0]), np.zeros(2))
    assert mo.tolist() == [0, 1] and counts.tolist() == [1, 1]  # test_score_dual.cpp:25-26
    assert abs(g - 0.8) <= 1e-12  # :49
    _, counts, mo = oracle.eval_dual(s, np.array([1.0, 1.0]), np.array([0.5, 0.0]))
    assert mo.tolist() == [1, 1] and counts.tolist() == [0, 2]  # :30-31
    r = oracle.solve_dual(s, np.array([1.0, 1.0]))
    assert abs(r["score"] - 0.8) <= 1e-9 and r["assignment"].tolist() == [0, 1]  # :76-78
    assert np.allclose(oracle.project_simplex([2.0, -1.0]), [1.0, 0.0])  # routing_opt:53-55
    prof = _table([[(0.0, 100.0), (10.0, 200.0)]])
    import ctypes as C
    pc = prof.c()
    at = lambda x: oracle.L.orc_latency_at(C.byref(pc), 0, C.c_double(x))  # noqa: E731
    assert at(5.0) == 150.0 and at(10.0) == 200.0 and at(0.0) == 100.0  # test_latency.cpp:91-93
    assert at(15.0) == 250.0  # :94


def test_invalid_targets_rejected(oracle):
    s = np.array([[0.9, 0.8], [0.4, 0.7]])
    with pytest.raises(ValueError):  # TargetCounts::validate (score_dual.cpp:195-205)
        oracle.solve_dual(s, np.array([1.0, 2.0]))


# ---- live pin against the compiled reference (skipped where oracle/_ref is absent) ----

def _synth(reference, n, m, seed):
    from paper_2604_10907_b200 import workloads as wl
    return reference.synth_scores(n, wl.beta_shapes(m), seed)


def test_synth_scores_host_matches_reference(reference):
    import paper_2604_10907_b200 as rw
    from paper_2604_10907_b200 import workloads as wl
    for n, m, seed in [(1, 1, 1), (777, 3, 9), (5000, 8, 1)]:
        ours = rw.synth_scores(n, [f"M{i}" for i in range(m)], wl.beta_shapes(m), seed).scores
        assert np.array_equal(bits(ours), bits(_synth(reference, n, m, seed)))


@pytest.mark.parametrize("n,m,kind", [(3000, 4, "int"), (2500, 5, "frac"), (1200, 8, "int"),
                                      (900, 16, "frac")])
def test_solve_dual_live(reference, oracle, n, m, kind):
    from oracle import Params
    s = _synth(reference, n, m, n + m)
    rng = np.random.default_rng(n)
    w = rng.dirichlet(np.full(m, 2.0))
    c = np.floor(w * n) if kind == "int" else n * w
    if kind == "int":
        c[0] += n - c.sum()
    p = Params(sub_max_iters=80)
    a = reference.solve_dual(s, c, p)
    b = oracle.solve_dual(s, c, p)
    assert np.array_equal(bits(a["alpha"]), bits(b["alpha"]))
    assert bits(a["score"]) == bits(b["score"])
    assert a["assignment"].tolist() == b["assignment"].tolist()


def test_select_setup_records_live(reference, oracle):
    """Every per-setup record of the reference select_setup equals the restatement's
    evaluate_setup (setup_search.cpp:187-211), and so does the winner (:246-253)."""
    from oracle import Params, ProfileTable
    from paper_2604_10907_b200 import workloads as wl
    cfg = wl.config("C1", n=800)
    inp = wl.build_inputs(cfg)
    s = wl.scores_for(cfg)
    tau = cfg.taus[0]
    p = Params(sub_max_iters=15, pga_max_iters=4, epsilon=(10.0 / tau) / 4)

    class Space:
        pass

    sp = Space()
    sp.tp_choices, sp.rho_choices = cfg.tp_choices, cfg.rho_choices
    sp.memory = [(cfg.models.index(mdl), tp, f) for (mdl, tp), f in cfg.mem.items()]
    sp.profile_keys = inp.profile_keys
    sp.profiles = ProfileTable(inp.koff, inp.kx, inp.ky)
    sp.gpu_count, sp.rho_floor = cfg.gpu_count, cfg.rho_floor
    sp.lambda_rps, sp.tau_ms, sp.kappa = cfg.lambda_rps, tau, cfg.kappa
    ref = reference.select_setup(s, sp, p, parallelism=4)
    assert ref["retained"] == len(inp.retained)
    assert ref["sweep_id"].tolist() == inp.retained.tolist()
    feas, sc, lat = [], [], []
    for k in range(len(inp.retained)):
        e = oracle.evaluate_setup(s, sp.profiles, inp.profile_index[k], cfg.lambda_rps, tau,
                                  cfg.kappa, p)
        assert bits(e["score"]) == bits(ref["sweep_score"][k])
        assert bits(e["latency_ms"]) == bits(ref["sweep_latency"][k])
        assert e["feasible"] == bool(ref["sweep_feasible"][k])
        feas.append(int(e["feasible"]))
        sc.append(e["score"])
        lat.append(e["latency_ms"])
    best = oracle.reduce(feas, sc, lat)
    assert ref["feasible"] == (best >= 0)
    if best >= 0:
        assert bits(ref["score"]) == bits(sc[best])


def test_enumerate_retain_host_matches_reference(reference):
    import paper_2604_10907_b200 as rw
    from paper_2604_10907_b200 import workloads as wl
    for name in ["C1", "C2", "C3"]:
        cfg = wl.config(name, n=10)

        class Space:
            pass

        sp = Space()
        sp.tp_choices, sp.rho_choices = cfg.tp_choices, cfg.rho_choices
        sp.memory = [(cfg.models.index(mdl), tp, f) for (mdl, tp), f in cfg.mem.items()]
        sp.gpu_count, sp.rho_floor = cfg.gpu_count, cfg.rho_floor
        ref_v, ref_tp, ref_rho = reference.enumerate_retain(sp)
        space = rw.SetupSpace(list(cfg.models), cfg.tp_choices, cfg.rho_choices)
        mem = rw.MemoryTable()
        for (mdl, tp), f in cfg.mem.items():
            mem.insert(mdl, tp, f)
        v, tp, rho = rw.enumerate_retain(space, cfg.gpu_count, cfg.rho_floor, mem)
        assert np.array_equal(v, ref_v) and np.array_equal(tp, ref_tp)
        assert np.array_equal(bits(rho), bits(ref_rho))
