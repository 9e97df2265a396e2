"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the checker libraries.

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement (oracle/rw_oracle.c).
* ``Reference`` -> oracle/_ref/libroutewise_ref.so, the unmodified reference library
  (/root/reference/proj/src, compiled by oracle/Makefile) behind oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference leg may
import this module.  The product (paper_2604_10907_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libroutewise_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def _l(a):
    return a.ctypes.data_as(_lp) if a is not None else None


class OrcSub(C.Structure):
    _fields_ = [("eta0", C.c_double), ("max_iters", C.c_int32), ("residual_tol", C.c_double),
                ("polish_passes", C.c_int32)]


class OrcPga(C.Structure):
    _fields_ = [("eta", C.c_double), ("max_iters", C.c_int32), ("w_tol", C.c_double),
                ("dual", OrcSub)]


class OrcBeta(C.Structure):
    _fields_ = [("beta_min", C.c_double), ("beta_max", C.c_double), ("epsilon", C.c_double),
                ("pga", OrcPga)]


class OrcCtx(C.Structure):
    _fields_ = [("lambda_rps", C.c_double), ("tau_ms", C.c_double), ("kappa", C.c_double)]


class OrcCounters(C.Structure):
    _fields_ = [("eval_passes", C.c_int64), ("polish_passes", C.c_int64),
                ("repair_calls", C.c_int64), ("solves", C.c_int64)]


class OrcProfiles(C.Structure):
    _fields_ = [("koff", _lp), ("kx", _dp), ("ky", _dp)]


class OrcRelaxed(C.Structure):
    _fields_ = [("objective", C.c_double), ("score", C.c_double), ("latency_ms", C.c_double),
                ("iterations", C.c_int32), ("converged", C.c_int32)]


class OrcBetaResult(C.Structure):
    _fields_ = [("feasible", C.c_int32), ("has_beta_star", C.c_int32), ("n_trace", C.c_int32),
                ("beta_star", C.c_double), ("best", OrcRelaxed)]


class OrcSetupEval(C.Structure):
    _fields_ = [("feasible", C.c_int32), ("score", C.c_double), ("latency_ms", C.c_double),
                ("beta", C.c_double)]


@dataclass
class Params:
    """Optimizer parameters (reference defaults, config.hpp:20-31)."""
    eta0: float = 1.0
    sub_max_iters: int = 500
    residual_tol: float = 1e-12
    polish_passes: int = 4
    pga_eta: float = 0.05
    pga_max_iters: int = 200
    w_tol: float = 1e-10
    beta_min: float = 0.0
    beta_max: float = -1.0
    epsilon: float = -1.0

    def sub(self):
        return OrcSub(self.eta0, self.sub_max_iters, self.residual_tol, self.polish_passes)

    def pga(self):
        return OrcPga(self.pga_eta, self.pga_max_iters, self.w_tol, self.sub())

    def beta(self):
        return OrcBeta(self.beta_min, self.beta_max, self.epsilon, self.pga())

    def pd(self):
        return np.array([self.pga_eta, self.w_tol, self.eta0, self.residual_tol], np.float64)

    def pi(self):
        return np.array([self.pga_max_iters, self.sub_max_iters, self.polish_passes], np.int32)


@dataclass
class ProfileTable:
    """CSR latency profiles: profile p has knots kx/ky[koff[p]:koff[p+1]]."""
    koff: np.ndarray
    kx: np.ndarray
    ky: np.ndarray

    @staticmethod
    def from_lists(knot_lists):
        koff = [0]
        kx, ky = [], []
        for knots in knot_lists:
            for x, y in knots:
                kx.append(float(x))
                ky.append(float(y))
            koff.append(len(kx))
        return ProfileTable(np.array(koff, np.int64), np.array(kx, np.float64),
                            np.array(ky, np.float64))

    def c(self):
        return OrcProfiles(_l(self.koff), _d(self.kx), _d(self.ky))


class Oracle:
    """The plain-C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        self.L = L
        L.orc_eval_dual.restype = C.c_double
        L.orc_latency_at.restype = C.c_double
        L.orc_latency_slope.restype = C.c_double
        L.orc_reduce.restype = C.c_int64

    def eval_dual(self, s, c, alpha, want_assign=True):
        n, m = s.shape
        counts = np.zeros(m, np.int32)
        mo = np.zeros(n, np.int32) if want_assign else None
        g = self.L.orc_eval_dual(n, m, _d(s), _d(c), _d(alpha), _i(counts), _i(mo), None)
        return g, counts, mo

    def solve_dual(self, s, c, p: Params = Params(), init_alpha=None):
        n, m = s.shape
        a = np.zeros(m)
        sc, db, gp = C.c_double(), C.c_double(), C.c_double()
        asg = np.zeros(n, np.int32)
        res = np.zeros(m)
        it, cv = C.c_int32(), C.c_int32()
        ctr = OrcCounters()
        sub = p.sub()
        ia = np.ascontiguousarray(init_alpha, np.float64) if init_alpha is not None else None
        rc = self.L.orc_solve_dual(n, m, _d(s), _d(np.ascontiguousarray(c, np.float64)),
                                   C.byref(sub), _d(ia), _d(a), C.byref(sc), C.byref(db),
                                   C.byref(gp), _i(asg), _d(res), C.byref(it), C.byref(cv),
                                   C.byref(ctr))
        if rc:
            raise ValueError("oracle solve_dual: invalid input")
        return dict(alpha=a, score=sc.value, dual_bound=db.value, gap=gp.value, assignment=asg,
                    residual=res, iterations=it.value, converged=bool(cv.value),
                    eval_passes=ctr.eval_passes, polish_passes=ctr.polish_passes,
                    repair_calls=ctr.repair_calls)

    def project_simplex(self, v):
        v = np.ascontiguousarray(v, np.float64)
        w = np.zeros_like(v)
        if self.L.orc_project_simplex(len(v), _d(v), _d(w)):
            raise ValueError("project_simplex: invalid input")
        return w

    def latency_eval(self, prof: ProfileTable, idx, w, lam, kappa):
        m = len(w)
        idx = np.ascontiguousarray(idx, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        lat = C.c_double()
        loads, lats = np.zeros(m), np.zeros(m)
        oor = np.zeros(m, np.int32)
        grad = np.zeros(m)
        pc = prof.c()
        self.L.orc_system_latency_eval(C.byref(pc), _i(idx), m, _d(w), C.c_double(lam),
                                       C.c_double(kappa), C.byref(lat), _d(loads), _d(lats),
                                       _i(oor))
        self.L.orc_system_latency_grad(C.byref(pc), _i(idx), m, _d(w), C.c_double(lam), _d(grad))
        return dict(latency=lat.value, loads=loads, lats=lats, oor=oor, grad=grad)

    def optimize_fractions(self, s, prof, idx, beta, lam, tau, kappa, p: Params = Params()):
        n, m = s.shape
        idx = np.ascontiguousarray(idx, np.int32)
        w = np.zeros(m)
        oor = np.zeros(m, np.int32)
        out = OrcRelaxed()
        ctr = OrcCounters()
        ctx = OrcCtx(lam, tau, kappa)
        pga = p.pga()
        pc = prof.c()
        rc = self.L.orc_optimize_fractions(n, m, _d(s), C.byref(pc), _i(idx), C.c_double(beta),
                                           C.byref(ctx), C.byref(pga), _d(w), _i(oor),
                                           C.byref(out), C.byref(ctr))
        if rc:
            raise ValueError("oracle optimize_fractions: invalid input")
        return dict(w=w, oor=oor, objective=out.objective, score=out.score,
                    latency_ms=out.latency_ms, iterations=out.iterations,
                    converged=bool(out.converged), eval_passes=ctr.eval_passes)

    def optimize_beta(self, s, prof, idx, lam, tau, kappa, p: Params = Params(), cap=256):
        n, m = s.shape
        idx = np.ascontiguousarray(idx, np.int32)
        w_star, best_w = np.zeros(m), np.zeros(m)
        best_oor = np.zeros(m, np.int32)
        out = OrcBetaResult()
        tb, ts, tl = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        tok = np.zeros(cap, np.int32)
        ctr = OrcCounters()
        ctx = OrcCtx(lam, tau, kappa)
        bp = p.beta()
        pc = prof.c()
        rc = self.L.orc_optimize_beta(n, m, _d(s), C.byref(pc), _i(idx), C.byref(ctx),
                                      C.byref(bp), _d(w_star), _d(best_w), _i(best_oor),
                                      C.byref(out), cap, _d(tb), _d(ts), _d(tl), _i(tok),
                                      C.byref(ctr))
        if rc:
            raise ValueError("oracle optimize_beta: invalid input")
        k = min(out.n_trace, cap)
        return dict(feasible=bool(out.feasible), has_beta_star=bool(out.has_beta_star),
                    beta_star=out.beta_star, w_star=w_star, best_w=best_w, best_oor=best_oor,
                    best_score=out.best.score, best_latency=out.best.latency_ms,
                    best_objective=out.best.objective, n_trace=out.n_trace,
                    trace_beta=tb[:k], trace_score=ts[:k], trace_latency=tl[:k],
                    trace_ok=tok[:k], eval_passes=ctr.eval_passes)

    def evaluate_setup(self, s, prof, idx, lam, tau, kappa, p: Params = Params()):
        n, m = s.shape
        idx = np.ascontiguousarray(idx, np.int32)
        out = OrcSetupEval()
        w = np.zeros(m)
        oor = np.zeros(m, np.int32)
        ctr = OrcCounters()
        ctx = OrcCtx(lam, tau, kappa)
        bp = p.beta()
        pc = prof.c()
        rc = self.L.orc_evaluate_setup(n, m, _d(s), C.byref(pc), _i(idx), C.byref(ctx),
                                       C.byref(bp), C.byref(out), _d(w), _i(oor), C.byref(ctr))
        if rc:
            raise ValueError("oracle evaluate_setup: invalid input")
        return dict(feasible=bool(out.feasible), score=out.score, latency_ms=out.latency_ms,
                    beta=out.beta, w=w, oor=oor, eval_passes=ctr.eval_passes,
                    polish_passes=ctr.polish_passes, repair_calls=ctr.repair_calls,
                    solves=ctr.solves)

    def reduce(self, feasible, score, latency):
        f = np.ascontiguousarray(feasible, np.int32)
        s = np.ascontiguousarray(score, np.float64)
        l = np.ascontiguousarray(latency, np.float64)
        return int(self.L.orc_reduce(len(f), _i(f), _d(s), _d(l)))


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Reference:
    """The unmodified reference library behind oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where "
                                    "/root/reference exists")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p

    def _chk(self, rc):
        if rc:
            raise RefError(rc, self.L.ref_last_error().decode())

    def synth_scores(self, n, shapes, seed):
        m = len(shapes)
        a = np.array([s[0] for s in shapes], np.float64)
        b = np.array([s[1] for s in shapes], np.float64)
        out = np.zeros((n, m), np.float64)
        self._chk(self.L.ref_synth_scores(n, m, _d(a), _d(b), C.c_uint64(seed), _d(out)))
        return out

    def dual_objective(self, s, c, alpha):
        n, m = s.shape
        g = C.c_double()
        self._chk(self.L.ref_dual_objective(n, m, _d(s), _d(np.asarray(c, np.float64)),
                                            _d(np.asarray(alpha, np.float64)), C.byref(g)))
        return g.value

    def assign_prompts(self, s, alpha):
        n, m = s.shape
        alpha = np.ascontiguousarray(alpha, np.float64)
        mo = np.zeros(n, np.int32)
        counts = np.zeros(m, np.int32)
        self._chk(self.L.ref_assign_prompts(n, m, _d(s), len(alpha), _d(alpha), _i(mo),
                                            _i(counts)))
        return mo, counts

    def solve_dual(self, s, c, p: Params = Params(), init_alpha=None):
        n, m = s.shape
        a = np.zeros(m)
        sc = np.zeros(3)
        asg = np.zeros(n, np.int32)
        res = np.zeros(m)
        oi = np.zeros(2, np.int32)
        ia = np.ascontiguousarray(init_alpha, np.float64) if init_alpha is not None else None
        self._chk(self.L.ref_solve_dual(n, m, _d(s), _d(np.ascontiguousarray(c, np.float64)),
                                        C.c_double(p.eta0), p.sub_max_iters,
                                        C.c_double(p.residual_tol), p.polish_passes, _d(ia),
                                        _d(a), _d(sc), _i(asg), _d(res), _i(oi)))
        return dict(alpha=a, score=sc[0], dual_bound=sc[1], gap=sc[2], assignment=asg,
                    residual=res, iterations=int(oi[0]), converged=bool(oi[1]))

    def exact_score_oracle(self, s, c, max_n=12):
        n, m = s.shape
        out = C.c_double()
        self._chk(self.L.ref_exact_score_oracle(n, m, _d(s), _d(np.asarray(c, np.float64)),
                                                max_n, C.byref(out)))
        return out.value

    def project_simplex(self, v):
        v = np.ascontiguousarray(v, np.float64)
        w = np.zeros_like(v)
        self._chk(self.L.ref_project_simplex(len(v), _d(v), _d(w)))
        return w

    def latency_at(self, knots, load):
        kx = np.array([k[0] for k in knots], np.float64)
        ky = np.array([k[1] for k in knots], np.float64)
        out, slope = C.c_double(), C.c_double()
        self._chk(self.L.ref_latency_at(len(knots), _d(kx), _d(ky), C.c_double(load),
                                        C.byref(out), C.byref(slope)))
        return out.value, slope.value

    def latency_eval(self, prof: ProfileTable, w, lam, kappa):
        """Single-setup evaluation: model i uses profile i."""
        m = len(w)
        w = np.ascontiguousarray(w, np.float64)
        lat = C.c_double()
        loads, lats, grad = np.zeros(m), np.zeros(m), np.zeros(m)
        oor = np.zeros(m, np.int32)
        self._chk(self.L.ref_system_latency_eval(m, _l(prof.koff), _d(prof.kx), _d(prof.ky),
                                                 _d(w), C.c_double(lam), C.c_double(kappa),
                                                 C.byref(lat), _d(loads), _d(lats), _i(oor),
                                                 _d(grad)))
        return dict(latency=lat.value, loads=loads, lats=lats, oor=oor, grad=grad)

    def optimize_fractions(self, s, prof, beta, lam, tau, kappa, p: Params = Params()):
        n, m = s.shape
        w = np.zeros(m)
        od = np.zeros(3)
        oi = np.zeros(2, np.int32)
        oor = np.zeros(m, np.int32)
        ctx = np.array([lam, tau, kappa], np.float64)
        self._chk(self.L.ref_optimize_fractions(n, m, _d(s), _l(prof.koff), _d(prof.kx),
                                                _d(prof.ky), _d(ctx), C.c_double(beta),
                                                _d(p.pd()), _i(p.pi()), _d(w), _d(od), _i(oi),
                                                _i(oor)))
        return dict(w=w, oor=oor, objective=od[0], score=od[1], latency_ms=od[2],
                    iterations=int(oi[0]), converged=bool(oi[1]))

    def optimize_beta(self, s, prof, lam, tau, kappa, p: Params = Params(), cap=256):
        n, m = s.shape
        w_star, best_w = np.zeros(m), np.zeros(m)
        best_oor = np.zeros(m, np.int32)
        od = np.zeros(4)
        oi = np.zeros(5, np.int32)
        tb, ts, tl = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        tok = np.zeros(cap, np.int32)
        ctx = np.array([lam, tau, kappa], np.float64)
        bp = np.array([p.beta_min, p.beta_max, p.epsilon], np.float64)
        self._chk(self.L.ref_optimize_beta(n, m, _d(s), _l(prof.koff), _d(prof.kx),
                                           _d(prof.ky), _d(ctx), _d(bp), _d(p.pd()),
                                           _i(p.pi()), _d(w_star), _d(best_w), _i(best_oor),
                                           _d(od), _i(oi), cap, _d(tb), _d(ts), _d(tl),
                                           _i(tok)))
        k = min(int(oi[4]), cap)
        return dict(feasible=bool(oi[0]), has_beta_star=bool(oi[1]), beta_star=od[0],
                    w_star=w_star, best_w=best_w, best_oor=best_oor, best_objective=od[1],
                    best_score=od[2], best_latency=od[3], n_trace=int(oi[4]),
                    trace_beta=tb[:k], trace_score=ts[:k], trace_latency=tl[:k],
                    trace_ok=tok[:k])

    def select_setup(self, s, space, p: Params = Params(), parallelism=0):
        """``space`` is a SweepSpace-like object (see tests/workloads.py)."""
        n, m = s.shape
        cap = int(np.prod([len(t) * len(r) for t, r in zip(space.tp_choices, space.rho_choices)]))
        tp_off = np.cumsum([0] + [len(t) for t in space.tp_choices]).astype(np.int32)
        tp_vals = np.array([x for t in space.tp_choices for x in t], np.int32)
        rho_off = np.cumsum([0] + [len(r) for r in space.rho_choices]).astype(np.int32)
        rho_vals = np.array([x for r in space.rho_choices for x in r], np.float64)
        mem = space.memory  # list of (model, tp, frac)
        mem_model = np.array([e[0] for e in mem], np.int32)
        mem_tp = np.array([e[1] for e in mem], np.int32)
        mem_frac = np.array([e[2] for e in mem], np.float64)
        pk = space.profile_keys  # list of (model, tp, rho), parallel to space.profiles CSR
        prof_model = np.array([k[0] for k in pk], np.int32)
        prof_tp = np.array([k[1] for k in pk], np.int32)
        prof_rho = np.array([k[2] for k in pk], np.float64)
        prof = space.profiles
        sp = np.array([space.gpu_count, space.rho_floor, space.lambda_rps, space.tau_ms,
                       space.kappa, p.beta_min, p.beta_max, p.epsilon, p.pga_eta, p.w_tol,
                       p.eta0, p.residual_tol], np.float64)
        si = np.array([p.pga_max_iters, p.sub_max_iters, p.polish_passes, parallelism],
                      np.int32)
        counts = np.zeros(3, np.int64)
        sw_id = np.zeros(cap, np.int64)
        sw_score, sw_lat = np.zeros(cap), np.zeros(cap)
        sw_feas = np.zeros(cap, np.int32)
        plan_d = np.zeros(3)
        plan_tp = np.zeros(m, np.int32)
        plan_rho, plan_w, plan_load = np.zeros(m), np.zeros(m), np.zeros(m)
        plan_oor = np.zeros(m, np.int32)
        self._chk(self.L.ref_select_setup(
            n, m, _d(s), _i(tp_off), _i(tp_vals), _i(rho_off), _d(rho_vals), len(mem),
            _i(mem_model), _i(mem_tp), _d(mem_frac), len(pk), _i(prof_model), _i(prof_tp),
            _d(prof_rho), _l(prof.koff), _d(prof.kx), _d(prof.ky), _d(sp), _i(si), _l(counts),
            cap, _l(sw_id), _d(sw_score), _d(sw_lat), _i(sw_feas), _d(plan_d), _i(plan_tp),
            _d(plan_rho), _d(plan_w), _d(plan_load), _i(plan_oor)))
        r = int(counts[1])
        return dict(enumerated=int(counts[0]), retained=r, feasible=bool(counts[2]),
                    sweep_id=sw_id[:r], sweep_score=sw_score[:r], sweep_latency=sw_lat[:r],
                    sweep_feasible=sw_feas[:r], score=plan_d[0], latency_ms=plan_d[1],
                    beta=plan_d[2], tp=plan_tp, rho=plan_rho, w=plan_w, load=plan_load,
                    oor=plan_oor)

    def enumerate_retain(self, space):
        m = len(space.tp_choices)
        cap = int(np.prod([len(t) * len(r) for t, r in zip(space.tp_choices, space.rho_choices)]))
        tp_off = np.cumsum([0] + [len(t) for t in space.tp_choices]).astype(np.int32)
        tp_vals = np.array([x for t in space.tp_choices for x in t], np.int32)
        rho_off = np.cumsum([0] + [len(r) for r in space.rho_choices]).astype(np.int32)
        rho_vals = np.array([x for r in space.rho_choices for x in r], np.float64)
        mem = space.memory
        mem_model = np.array([e[0] for e in mem], np.int32)
        mem_tp = np.array([e[1] for e in mem], np.int32)
        mem_frac = np.array([e[2] for e in mem], np.float64)
        n_enum = C.c_int64()
        verdict = np.zeros(cap, np.int32)
        tp_out = np.zeros((cap, m), np.int32)
        rho_out = np.zeros((cap, m), np.float64)
        self._chk(self.L.ref_enumerate_retain(
            m, _i(tp_off), _i(tp_vals), _i(rho_off), _d(rho_vals), len(mem), _i(mem_model),
            _i(mem_tp), _d(mem_frac), int(space.gpu_count), C.c_double(space.rho_floor),
            C.c_int64(cap), C.byref(n_enum), _i(verdict), _i(tp_out), _d(rho_out)))
        return verdict, tp_out, rho_out
