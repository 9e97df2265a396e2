"""BASELINE.md's parity protocol on the GPU, against the UNMODIFIED reference.

Fixtures (tests/golden/protocol_*.json, made by tests/golden/gen_protocol.py through
oracle/_ref's select_setup and solve_dual): full N, the first 64 retained setups, the
truncated schedule — C2 at all 8 SLOs, C3 (1M x 8), C5 (1M x 8 adversarial ties) — and one
default-schedule sweep (C1 shape, N = 2000, all 64 setups, config.hpp:20-31).

Every record is compared bit for bit: feasible, score and latency against the reference's
sweep rows (setup_search.cpp:187-211), beta, w and the pass counters against the pinned C
restatement; the winner against the reference's plan (setup_search.cpp:246-253); and the
winner's routing policy {alpha*, counts, assignment} against the reference's
solve_dual(N * w*) (test_cli.cpp:103-106).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2604_10907_b200 as rw
from paper_2604_10907_b200 import workloads as wl

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    path = os.path.join(GOLD, f"protocol_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    with open(path) as f:
        return json.load(f)


def hb(h):
    """hex float -> int64 bit pattern"""
    return np.float64(float.fromhex(h)).view(np.int64)


def bits(x):
    return np.asarray(x, np.float64).view(np.int64)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def schedule(g, tau):
    if g["schedule"] == "default":
        return rw.BetaSearchParams(), rw.SubgradientParams()
    p = wl.with_span_epsilon(wl.truncated_params(), tau, 4.0)
    return p, p.pga.dual


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2", "C3", "C5", "C1D"])
def test_protocol_vs_reference(eng, name):
    g = load(name)
    cfg = wl.config(g["config"], g["n"])
    inp = wl.build_inputs(cfg)
    s = wl.scores_for(cfg)
    assert sha(s) == g["scores_sha256"], "inputs differ from the fixture's"
    m = cfg.m
    eng.load_scores(s)
    eng.load_profiles(inp.koff, inp.kx, inp.ky)
    S = g["slos"][0]["setups"]
    taus = [sl["tau"] for sl in g["slos"]]
    params = [schedule(g, t)[0] for t in taus]
    for p, sl in zip(params, g["slos"]):
        assert bits(p.epsilon) == hb(sl["params"]["epsilon"]) or g["schedule"] == "default"
    opt = rw.OptimizeContext(lambda_rps=cfg.lambda_rps, tau_ms=taus[0], kappa=cfg.kappa)
    recs = eng.sweep_slo(inp.profile_index[:S], inp.retained[:S], taus, opt, params)
    assert len(recs) == S * len(taus)
    for ti, sl in enumerate(g["slos"]):
        part = recs[ti * S:(ti + 1) * S]
        for k in range(S):
            r, ref = part[k], sl["sweep"][k]
            assert int(r["setup_id"]) == ref["id"] and int(r["status"]) == 0
            assert bool(r["feasible"]) == ref["feasible"], (name, sl["tau"], k)
            assert bits(r["score"]) == hb(ref["score"]), (name, sl["tau"], k)
            assert bits(r["latency_ms"]) == hb(ref["latency_ms"]), (name, sl["tau"], k)
            assert 0 < int(r["exec_passes"]) <= int(r["eval_passes"])
            if sl["oracle"] is None:  # C5: rows, plan and policy from the reference only
                continue
            orc = sl["oracle"][k]
            assert bits(r["beta"]) == hb(orc["beta"]), (name, sl["tau"], k)
            assert np.array_equal(bits(r["w"][:m]), [hb(x) for x in orc["w"]]), (name, k)
            assert int(r["eval_passes"]) == orc["eval_passes"], (name, sl["tau"], k)
            assert int(r["polish_passes"]) == orc["polish_passes"], (name, sl["tau"], k)
            assert int(r["repair_calls"]) == orc["repair_calls"], (name, sl["tau"], k)
        win = rw.reduce_records(part)
        plan = sl["plan"]
        assert (win if win >= 0 else None) == plan["winner"], (name, sl["tau"])
        if win < 0:
            continue
        w = part[win]
        assert bits(w["score"]) == hb(plan["score"])
        assert bits(w["latency_ms"]) == hb(plan["latency_ms"])
        assert bits(w["beta"]) == hb(plan["beta"])
        assert np.array_equal(bits(w["w"][:m]), [hb(x) for x in plan["w"]])
        # the winner's routing policy: bit-exact alpha*, counts and assignment
        _, sub = schedule(g, sl["tau"])
        ds, asg = eng.winner_policy(w["w"][:m], sub)
        pol = sl["policy"]
        assert np.array_equal(bits(ds.alpha_star.alpha), [hb(x) for x in pol["alpha"]])
        assert bits(ds.score) == hb(pol["score"])
        assert bits(ds.dual_bound) == hb(pol["dual_bound"])
        assert list(ds.counts) == pol["counts"]
        assert sha(asg.astype(np.int32)) == pol["assignment_sha256"]
