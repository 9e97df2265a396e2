"""GPU parity: the sm_100a path vs the reference (oracle/_ref) and the C restatement, on
seeded inputs.  Bar: bit-exact — g bits, counts, assignments, prices, scores,
latencies, pass counts."""
import numpy as np
import pytest

import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def bits(x):
    return np.asarray(x, np.float64).view(np.int64)


def synth(n, m, seed=1):
    return rw.synth_scores(n, [f"M{i}" for i in range(m)], wl.beta_shapes(m), seed).scores


@pytest.mark.parametrize("n,m", [(1, 1), (2, 2), (17, 3), (1000, 4), (4096, 4), (4097, 5),
                                 (10000, 4), (100003, 8), (30000, 16), (5000, 32),
                                 (20000, 13)])
def test_eval_pass_bit_exact(eng, oracle, n, m):
    s = synth(n, m, seed=n + m)
    eng.load_scores(s)
    rng = np.random.default_rng(n * 31 + m)
    c = np.full(m, n / m)
    for alpha in [np.zeros(m), rng.uniform(-1, 1, m), rng.uniform(0, 0.3, m),
                  rng.uniform(2, 3, m), -rng.uniform(2, 3, m), rng.uniform(-1e-3, 1e-3, m)]:
        g = eng.dual_objective(c, alpha)
        mo, counts = eng.assign_prompts(alpha)
        g_ref, counts_ref, mo_ref = oracle.eval_dual(s, c, alpha)
        assert bits(g) == bits(g_ref), (alpha, g, g_ref)
        assert np.array_equal(counts, counts_ref)
        assert np.array_equal(mo, mo_ref)


def test_eval_pass_ties(eng, oracle):
    s = wl.tie_scores(synth(50000, 8, 3), 3)
    eng.load_scores(s)
    m = 8
    c = np.full(m, 50000 / m)
    for alpha in [np.zeros(m), np.arange(m) / 16.0, np.full(m, 0.25)]:
        g = eng.dual_objective(c, alpha)
        mo, counts = eng.assign_prompts(alpha)
        g_ref, counts_ref, mo_ref = oracle.eval_dual(s, c, alpha)
        assert bits(g) == bits(g_ref)
        assert np.array_equal(counts, counts_ref) and np.array_equal(mo, mo_ref)


def test_worked_examples(eng):
    # test_score_dual.cpp:21-39, 46-55
    s = np.array([[0.9, 0.8], [0.4, 0.7]])
    eng.load_scores(s)
    mo, counts = eng.assign_prompts([0.0, 0.0])
    assert mo.tolist() == [0, 1] and counts.tolist() == [1, 1]
    mo, counts = eng.assign_prompts([0.5, 0.0])
    assert mo.tolist() == [1, 1] and counts.tolist() == [0, 2]
    assert abs(eng.dual_objective([1.0, 1.0], [0.0, 0.0]) - 0.8) <= 1e-12
    assert abs(eng.dual_objective([1.0, 1.0], [0.1, 0.1]) - 0.8) <= 1e-12
    sol = eng.solve_dual([1.0, 1.0])
    assert abs(sol.score - 0.8) <= 1e-9 and sol.assignment == [0, 1]
    assert min(sol.alpha_star.alpha) == 0.0
    eng.load_scores(np.array([[0.5, 0.5]]))
    assert eng.assign_prompts([0.0, 0.0])[0].tolist() == [0]
    eng.load_scores(np.array([[0.3, 0.7, 0.7]]))
    assert eng.assign_prompts([0.0, 0.0, 0.0])[0].tolist() == [1]


def _cmp_solution(got, ref):
    assert bits(got.score) == bits(ref["score"]), (got.score, ref["score"])
    assert bits(got.dual_bound) == bits(ref["dual_bound"])
    assert bits(got.duality_gap) == bits(ref["gap"])
    assert np.array_equal(bits(got.alpha_star.alpha), bits(ref["alpha"]))
    assert np.array_equal(bits(got.count_residual), bits(ref["residual"]))
    assert got.assignment == ref["assignment"].tolist()
    assert got.iterations == ref["iterations"] and got.converged == ref["converged"]


@pytest.mark.parametrize("n,m,kind", [(8, 2, "int"), (40, 3, "frac"), (1000, 4, "int"),
                                      (1000, 4, "frac"), (10000, 4, "int"),
                                      (10000, 4, "frac"), (12000, 8, "int"),
                                      (6000, 16, "frac"), (3000, 5, "int")])
def test_solve_dual_bit_exact(eng, reference, oracle, n, m, kind):
    s = synth(n, m, seed=7 * n + m)
    eng.load_scores(s)
    rng = np.random.default_rng(n + 3 * m)
    w = rng.dirichlet(np.full(m, 2.0))
    if kind == "int":
        c = np.floor(w * n)
        c[0] += n - c.sum()
    else:
        c = n * w
    p = rw.SubgradientParams(max_iters=120)
    from oracle import Params
    rp_ = Params(sub_max_iters=120)
    got = eng.solve_dual(c, p)
    ref = reference.solve_dual(s, c, rp_)
    _cmp_solution(got, ref)
    orc = oracle.solve_dual(s, c, rp_)
    assert got.eval_passes == orc["eval_passes"]
    # warm start
    init = rng.uniform(0, 0.2, m)
    got = eng.solve_dual(c, p, init)
    ref = reference.solve_dual(s, c, rp_, init_alpha=init)
    _cmp_solution(got, ref)


def _profiles(m):
    from oracle import ProfileTable
    return ProfileTable.from_lists([wl.linear_knots(i, 1, 1.0) for i in range(m)])


@pytest.mark.parametrize("n,m,beta", [(500, 2, 0.01), (3000, 4, 0.05), (2000, 3, 0.0)])
def test_optimize_fractions_bit_exact(eng, reference, n, m, beta):
    from oracle import Params
    s = synth(n, m, seed=n)
    prof = _profiles(m)
    eng.load_scores(s)
    eng.load_profiles(prof.koff, prof.kx, prof.ky)
    p = Params(sub_max_iters=60, pga_max_iters=12)
    opt = rw.OptimizeContext(lambda_rps=40.0, tau_ms=120.0, kappa=1.25)
    pga = rw.PgaParams(0.05, 12, 1e-10, rw.SubgradientParams(1.0, 60, 1e-12, 4))
    got = eng.optimize_fractions(np.arange(m), beta, opt, pga)
    ref = reference.optimize_fractions(s, prof, beta, 40.0, 120.0, 1.25, p)
    assert np.array_equal(bits(got.w.w), bits(ref["w"]))
    assert bits(got.score) == bits(ref["score"])
    assert bits(got.latency_ms) == bits(ref["latency_ms"])
    assert bits(got.objective) == bits(ref["objective"])
    assert got.iterations == ref["iterations"] and got.converged == ref["converged"]
    assert got.out_of_range == [bool(x) for x in ref["oor"]]


@pytest.mark.parametrize("n,m,tau", [(2000, 4, 120.0), (1500, 3, 60.0), (800, 2, 400.0)])
def test_optimize_beta_bit_exact(eng, reference, n, m, tau):
    from oracle import Params
    s = synth(n, m, seed=n + 1)
    prof = _profiles(m)
    eng.load_scores(s)
    eng.load_profiles(prof.koff, prof.kx, prof.ky)
    p = Params(sub_max_iters=40, pga_max_iters=6)
    opt = rw.OptimizeContext(lambda_rps=40.0, tau_ms=tau, kappa=1.25)
    bp = rw.BetaSearchParams(0.0, -1.0, -1.0,
                             rw.PgaParams(0.05, 6, 1e-10, rw.SubgradientParams(1.0, 40, 1e-12, 4)))
    got = eng.optimize_beta(np.arange(m), opt, bp)
    ref = reference.optimize_beta(s, prof, 40.0, tau, 1.25, p)
    assert got.feasible == ref["feasible"]
    assert len(got.trace) == ref["n_trace"]
    for st, b, sc, lt, ok in zip(got.trace, ref["trace_beta"], ref["trace_score"],
                                 ref["trace_latency"], ref["trace_ok"]):
        assert bits(st.beta) == bits(b) and bits(st.score) == bits(sc)
        assert bits(st.latency_ms) == bits(lt) and st.feasible == bool(ok)
    if got.feasible:
        assert bits(got.beta_star) == bits(ref["beta_star"])
        assert np.array_equal(bits(got.best.w.w), bits(ref["best_w"]))
        assert bits(got.best.score) == bits(ref["best_score"])


def test_sweep_c1_truncated_vs_oracle(eng, oracle):
    """C1 shape (10k x 4 x 64 setups) on a truncated schedule: every record bit-exact."""
    from oracle import Params, ProfileTable
    cfg = wl.config("C1")
    inp = wl.build_inputs(cfg)
    s = wl.scores_for(cfg)
    eng.load_scores(s)
    eng.load_profiles(inp.koff, inp.kx, inp.ky)
    tau = cfg.taus[0]
    bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
    recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
    assert len(recs) == len(inp.retained) == 64
    prof = ProfileTable(inp.koff, inp.kx, inp.ky)
    p = Params(sub_max_iters=20, pga_max_iters=5, epsilon=bp.epsilon)
    for r, k in zip(recs, range(len(inp.retained))):
        ref = oracle.evaluate_setup(s, prof, inp.profile_index[k], cfg.lambda_rps, tau,
                                    cfg.kappa, p)
        assert int(r["setup_id"]) == int(inp.retained[k])
        assert bool(r["feasible"]) == ref["feasible"]
        assert bits(r["score"]) == bits(ref["score"]), (k, float(r["score"]), ref["score"])
        assert bits(r["latency_ms"]) == bits(ref["latency_ms"])
        assert bits(r["beta"]) == bits(ref["beta"])
        assert int(r["eval_passes"]) == ref["eval_passes"]


def test_sweep_slo_batch_matches_single_slo(eng, oracle):
    """(setup, tau) batching: records equal per-SLO sweeps and the C oracle."""
    from oracle import Params, ProfileTable
    cfg = wl.config("C2", n=3000)
    inp = wl.build_inputs(cfg, limit=24)
    s = wl.scores_for(cfg)
    eng.load_scores(s)
    eng.load_profiles(inp.koff, inp.kx, inp.ky)
    taus = [60.0, 120.0, 250.0]
    params = [wl.with_span_epsilon(wl.truncated_params(), t, 4.0) for t in taus]
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=0.0, kappa=cfg.kappa)
    recs = eng.sweep_slo(inp.profile_index, inp.retained, taus, opt, params)
    S = len(inp.retained)
    assert len(recs) == S * len(taus)
    prof = ProfileTable(inp.koff, inp.kx, inp.ky)
    for ti, (t, p) in enumerate(zip(taus, params)):
        one = eng.sweep(inp.profile_index, inp.retained,
                        rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=t, kappa=cfg.kappa), p)
        part = recs[ti * S:(ti + 1) * S]
        assert np.array_equal(part["score"].view(np.int64), one["score"].view(np.int64))
        assert np.array_equal(part["setup_id"], one["setup_id"])
        assert (part["tau_ms"] == t).all()
        op = Params(sub_max_iters=20, pga_max_iters=5, epsilon=p.epsilon)
        for k in range(0, S, 7):
            ref = oracle.evaluate_setup(s, prof, inp.profile_index[k], cfg.lambda_rps, t,
                                        cfg.kappa, op)
            assert bits(part[k]["score"]) == bits(ref["score"])
            assert bits(part[k]["latency_ms"]) == bits(ref["latency_ms"])
            assert int(part[k]["eval_passes"]) == ref["eval_passes"]


@pytest.mark.parametrize("name,n,limit", [("C3", 20000, 6), ("C5", 20000, 6), ("C4", 6000, 3)])
def test_sweep_configs_reduced_vs_oracle(eng, oracle, name, n, limit):
    """Configs C3 (8 models incl. TP), C5 (adversarial ties: quantised scores, duplicated
    columns, 1-ulp neighbours) and C4 (16 models, nonlinear 12-knot latency) at reduced N:
    every record bit-exact vs the C restatement, pass counts included."""
    from oracle import Params, ProfileTable
    cfg = wl.config(name, n=n)
    inp = wl.build_inputs(cfg, limit=limit)
    s = wl.scores_for(cfg)
    eng.load_scores(s)
    eng.load_profiles(inp.koff, inp.kx, inp.ky)
    tau = cfg.taus[0]
    bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
    recs = eng.sweep(inp.profile_index, inp.retained, opt, bp)
    prof = ProfileTable(inp.koff, inp.kx, inp.ky)
    p = Params(sub_max_iters=20, pga_max_iters=5, epsilon=bp.epsilon)
    for k, r in enumerate(recs):
        ref = oracle.evaluate_setup(s, prof, inp.profile_index[k], cfg.lambda_rps, tau,
                                    cfg.kappa, p)
        assert bool(r["feasible"]) == ref["feasible"], k
        assert bits(r["score"]) == bits(ref["score"]), (k, float(r["score"]), ref["score"])
        assert bits(r["latency_ms"]) == bits(ref["latency_ms"]), k
        assert bits(r["beta"]) == bits(ref["beta"]), k
        assert np.array_equal(bits(r["w"][:cfg.m]), bits(ref["w"])), k
        assert int(r["eval_passes"]) == ref["eval_passes"], k


@pytest.mark.parametrize("name", ["C3", "C5", "C4"])
def test_eval_pass_full_size_vs_oracle(eng, oracle, name):
    """BASELINE sizes (1M x 8, 10M x 16): one priced pass and the final assignment, bit
    for bit."""
    cfg = wl.config(name)
    s = wl.scores_for(cfg)
    eng.load_scores(s)
    m = cfg.m
    c = np.full(m, cfg.n / m)
    rng = np.random.default_rng(5)
    for alpha in [np.zeros(m), rng.uniform(-0.05, 0.05, m), np.arange(m) / 16.0]:
        g = eng.dual_objective(c, alpha)
        mo, counts = eng.assign_prompts(alpha)
        g_ref, counts_ref, mo_ref = oracle.eval_dual(s, c, alpha)
        assert bits(g) == bits(g_ref)
        assert np.array_equal(counts, counts_ref) and np.array_equal(mo, mo_ref)


def _solve_vs_oracle(eng, oracle, s, c, sub_iters=20):
    from oracle import Params
    eng.load_scores(s)
    got = eng.solve_dual(c, rw.SubgradientParams(1.0, sub_iters, 1e-12, 4))
    ref = oracle.solve_dual(s, c, Params(sub_max_iters=sub_iters))
    assert np.array_equal(bits(got.alpha_star.alpha), bits(ref["alpha"]))
    assert bits(got.score) == bits(ref["score"]), (got.score, ref["score"])
    assert bits(got.dual_bound) == bits(ref["dual_bound"])
    assert np.array_equal(np.asarray(got.assignment), ref["assignment"])
    assert got.eval_passes == ref["eval_passes"]
    return got, ref


@pytest.mark.parametrize("n", [30_000, 100_000])
def test_solve_dual_c5_ties_repair_vs_oracle(eng, oracle, n):
    """C5's adversarial ties at integral targets: repair Phase 2 runs thousands of cycles
    (score_dual.cpp:120-180) — the incremental pair lists must pick the same witnesses in
    the same order as the reference's full re-sweeps."""
    cfg = wl.config("C5", n=n)
    s = wl.scores_for(cfg)
    c = np.full(cfg.m, n / cfg.m)
    _solve_vs_oracle(eng, oracle, s, c)


def test_polish_tie_group_larger_than_candidate_buffer(eng, oracle):
    """more than 4096 rows share the k-th largest b of a polish coordinate (the
    overfull-shell narrowing ends on one key value): the answer is that value."""
    n = 20_000
    rng = np.random.default_rng(3)
    s = np.empty((n, 2))
    s[:, 0] = 0.5
    s[:, 1] = 0.25
    s[18_000:, 1] = rng.uniform(0.0, 1.0, n - 18_000)
    for c in ([10_000.0, 10_000.0], [4_000.0, 16_000.0], [9_999.5, 10_000.5]):
        _solve_vs_oracle(eng, oracle, s, np.array(c))


def test_binary_file_and_pinned_async_load_give_identical_sweeps(eng, tmp_path):
    """f2: scores through a .f64 file and a page-locked host buffer (rw_load_scores enqueues
    the H2D and returns) give the same records as the in-memory path."""
    import torch
    from paper_2604_10907_b200 import routeplan as rp
    cfg = wl.config("C2", n=20000)
    inp = wl.build_inputs(cfg, limit=8)
    s = wl.scores_for(cfg)
    path = str(tmp_path / "c2.f64")
    rp.write_scores_f64(rp.ScoreMatrix([f"p{j + 1}" for j in range(cfg.n)], cfg.models, s), path)
    t = rp.read_scores_f64(path).scores
    pinned = torch.from_numpy(t).pin_memory().numpy()
    tau = cfg.taus[3]
    bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
    out = []
    for src in (s, pinned):
        eng.load_scores(src)
        eng.load_profiles(inp.koff, inp.kx, inp.ky)
        out.append(eng.sweep(inp.profile_index, inp.retained, opt, bp))
    assert out[0].tobytes() == out[1].tobytes()


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_speculative_bisection_records_identical(eng, depth):
    """f4: rw_sweep_spec evaluates `depth` levels of each instance's beta-bisection tree per
    launch and follows the realised path on the host (routing_opt.cpp:154-171) — every
    record field equals the sequential sweep's, bit for bit, except exec_passes (which also
    counts the discarded speculative branches)."""
    cfg = wl.config("C1", n=3000)
    inp = wl.build_inputs(cfg)
    s = wl.scores_for(cfg)
    eng.load_scores(s)
    eng.load_profiles(inp.koff, inp.kx, inp.ky)
    taus = [90.0, 120.0]
    params = [wl.with_span_epsilon(wl.truncated_params(), t, 16.0) for t in taus]
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=taus[0], kappa=cfg.kappa)
    seq = eng.sweep_slo(inp.profile_index, inp.retained, taus, opt, params)
    spec = eng.sweep_spec(inp.profile_index, inp.retained, taus, opt, params, depth=depth)
    assert len(seq) == len(spec) == 128
    for f in seq.dtype.names:
        if f == "exec_passes":
            assert (spec[f] > 0).all()  # memo hits depend on which CTA ran what
            continue
        assert np.ascontiguousarray(seq[f]).tobytes() == np.ascontiguousarray(spec[f]).tobytes(), f
    assert (seq["bisect_steps"] >= 3).all()  # span/16: a real bisection


def test_sweep_async_returns_before_the_kernel_and_stages_its_tables(eng):
    """rw_sweep_slo_async enqueues the launch and returns without waiting for the device,
    and the setup / SLO tables it was given may change as soon as it returns (they are
    staged through a context-owned host buffer): the records equal the blocking sweep's."""
    import time
    cfg = wl.config("C2", n=100_000)
    inp = wl.build_inputs(cfg, limit=64)
    eng.load_scores(wl.scores_for(cfg))
    eng.load_profiles(inp.koff, inp.kx, inp.ky)
    tau = cfg.taus[0]
    bp = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=tau, kappa=cfg.kappa)
    ref = eng.sweep(inp.profile_index, inp.retained, opt, bp)
    kernel_ms = eng.last_kernel_ms()
    t0 = time.perf_counter()
    eng.sweep_async(inp.profile_index, inp.retained, opt, bp)
    call_ms = (time.perf_counter() - t0) * 1e3
    _, ids, taus, _, _, _ = eng._pending
    ids[:] = 0          # the caller reuses its buffers right away
    taus[:] = 1.0
    recs = eng.sweep_fetch()
    for f in ref.dtype.names:
        if f == "exec_passes":  # memo hits depend on which CTA ran what
            continue
        assert np.ascontiguousarray(recs[f]).tobytes() == np.ascontiguousarray(ref[f]).tobytes(), f
    assert kernel_ms > 50.0, kernel_ms  # a launch long enough for the timing to mean something
    assert call_ms < 0.5 * kernel_ms, (call_ms, kernel_ms)
