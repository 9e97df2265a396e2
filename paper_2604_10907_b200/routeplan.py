"""Host-side mirror of the reference C++ solver API (routeplan::*), over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/routeplan/
(score_dual.hpp, latency.hpp, routing_opt.hpp, setup_search.hpp, types.hpp,
workload.hpp), so parity tests read like the reference's own doctest cases.  Every solver
call runs the sm_100a kernels in librw_b200.so; nothing here computes a result on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from ._abi import dptr, iptr, lptr

# ---------------------------------------------------------------------------------------
# errors (errors.hpp:9-18)


class ValidationError(RuntimeError):
    """Bad data: out-of-range values, dimension mismatches."""


class ConfigError(RuntimeError):
    """Bad wiring: missing profile / memory keys."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the B200 path."""


def _raise(code: int, msg: str):
    if code == _abi.RW_ERR_VALIDATION:
        raise ValidationError(msg)
    if code == _abi.RW_ERR_CONFIG:
        raise ConfigError(msg)
    if code == _abi.RW_ERR_UNSUPPORTED:
        raise ValidationError(msg)
    raise DeviceError(msg)


def format_double(v: float) -> str:
    """Shortest round-trip text (csv.cpp:78-84 uses std::to_chars)."""
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") else r


# ---------------------------------------------------------------------------------------
# types (types.hpp, workload.hpp, score_dual.hpp, latency.hpp, routing_opt.hpp)


class Metric(enum.IntEnum):
    TTFT = 0
    TPOT = 1
    E2E = 2


def parse_metric(name: str) -> Metric:
    try:
        return Metric[name]
    except KeyError:
        raise ValidationError(f"unknown metric '{name}' (expected TTFT, TPOT, or E2E)") from None


@dataclass
class ScoreMatrix:
    """Dense prompt-by-model scores, row-major N x M (workload.hpp:12-23)."""
    prompts: List[str]
    models: List[str]
    scores: np.ndarray

    def n(self):
        return len(self.prompts)

    def m(self):
        return len(self.models)

    def at(self, j, i):
        return float(self.scores[j, i])

    @staticmethod
    def from_array(a, models=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        n, m = a.shape
        models = models or [chr(ord("A") + i) if m <= 26 else f"M{i}" for i in range(m)]
        return ScoreMatrix([f"p{j + 1}" for j in range(n)], list(models), a)


@dataclass
class TargetCounts:
    counts: List[float]

    def m(self):
        return len(self.counts)


@dataclass
class DualPrices:
    alpha: List[float]

    def m(self):
        return len(self.alpha)


@dataclass
class Assignment:
    model_of: List[int]
    counts: List[int]


@dataclass
class SubgradientParams:
    eta0: float = 1.0
    max_iters: int = 500
    residual_tol: float = 1e-12
    polish_passes: int = 4
    init_alpha: List[float] = field(default_factory=list)

    def c(self):
        return _abi.rw_subgradient_params(self.eta0, self.max_iters, self.residual_tol,
                                          self.polish_passes)


@dataclass
class DualSolution:
    alpha_star: DualPrices
    score: float
    dual_bound: float
    duality_gap: float
    assignment: List[int]
    count_residual: List[float]
    iterations: int
    converged: bool
    counts: List[int] = field(default_factory=list)
    eval_passes: int = 0


@dataclass
class LatencyProfile:
    model: str
    tp: int
    rho: float
    metric: Metric
    knots: List[Tuple[float, float]]

    def max_measured_load(self):
        return self.knots[-1][0]

    def validate(self):
        who = f"profile {describe_profile_key(self.model, self.tp, self.rho, self.metric)}"
        if len(self.knots) < 2:
            raise ValidationError(f"{who}: needs at least two knots")
        for k, (x, y) in enumerate(self.knots):
            if x < 0.0 or y < 0.0:
                raise ValidationError(f"{who}: negative load or latency")
            if k > 0 and not (x > self.knots[k - 1][0]):
                raise ValidationError(f"{who}: loads must be strictly increasing")


def quantize_rho(rho: float) -> int:
    # latency.cpp:12 std::lround(rho * 1e4): half away from zero
    x = rho * 1e4
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def describe_profile_key(model, tp, rho, metric) -> str:
    return (f"(model={model}, tp={tp}, rho={format_double(rho)}, "
            f"metric={Metric(metric).name})")


class ProfileLibrary:
    """(model, tp, round(rho*1e4), metric) -> LatencyProfile (latency.hpp:36-42)."""

    def __init__(self):
        self.profiles: Dict[tuple, LatencyProfile] = {}

    def add(self, p: LatencyProfile):
        self.profiles[(p.model, p.tp, quantize_rho(p.rho), int(p.metric))] = p

    def contains(self, model, tp, rho, metric) -> bool:
        return (model, tp, quantize_rho(rho), int(metric)) in self.profiles

    def at(self, model, tp, rho, metric) -> LatencyProfile:
        key = (model, tp, quantize_rho(rho), int(metric))
        if key not in self.profiles:
            raise ConfigError(
                f"no latency profile for {describe_profile_key(model, tp, rho, metric)}")
        return self.profiles[key]


@dataclass
class ModelSetup:
    model: str
    tp: int = 1
    rho: float = 1.0


@dataclass
class SystemSetup:
    per_model: List[ModelSetup]

    def m(self):
        return len(self.per_model)

    def validate(self):  # types.cpp:27-38
        if not self.per_model:
            raise ValidationError("setup: no models")
        seen = set()
        for ms in self.per_model:
            if not ms.model:
                raise ValidationError("setup: empty model name")
            if ms.model in seen:
                raise ValidationError(f"setup: duplicate model '{ms.model}'")
            seen.add(ms.model)
            if ms.tp < 1:
                raise ValidationError(f"setup: model '{ms.model}' tp must be >= 1")
            if not (ms.rho > 0.0) or ms.rho > 1.0:
                raise ValidationError(f"setup: model '{ms.model}' rho must lie in (0, 1]")


class MemoryTable:
    """Per-(model, tp) shard memory fraction (types.hpp:33-48)."""

    def __init__(self):
        self.entries: Dict[Tuple[str, int], float] = {}

    def insert(self, model, tp, frac):
        if (model, tp) in self.entries:
            raise ValidationError(f"memory table: duplicate entry for ({model}, tp={tp})")
        self.entries[(model, tp)] = float(frac)

    def contains(self, model, tp):
        return (model, tp) in self.entries

    def at(self, model, tp):
        if (model, tp) not in self.entries:
            raise ConfigError(f"memory table: no entry for ({model}, tp={tp})")
        return self.entries[(model, tp)]


@dataclass
class RoutingFractions:
    w: List[float]

    def m(self):
        return len(self.w)


@dataclass
class OptimizeContext:
    scores: Optional[ScoreMatrix] = None
    lib: Optional[ProfileLibrary] = None
    lambda_rps: float = 0.0
    tau_ms: float = 0.0
    metric: Metric = Metric.TTFT
    kappa: float = 1.25

    def c(self):
        return _abi.rw_opt_context(self.lambda_rps, self.tau_ms, self.kappa)


@dataclass
class PgaParams:
    eta: float = 0.05
    max_iters: int = 200
    w_tol: float = 1e-10
    dual: SubgradientParams = field(default_factory=SubgradientParams)
    on_iterate: Optional[Callable] = None  # not supported on device (no host round trip)

    def c(self):
        return _abi.rw_pga_params(self.eta, self.max_iters, self.w_tol, self.dual.c())


@dataclass
class RelaxedSolveResult:
    w: RoutingFractions
    objective: float
    score: float
    latency_ms: float
    iterations: int
    converged: bool
    out_of_range: List[bool]
    eval_passes: int = 0


@dataclass
class BetaStep:
    beta: float
    score: float
    latency_ms: float
    feasible: bool


@dataclass
class BetaSearchParams:
    beta_min: float = 0.0
    beta_max: float = -1.0
    epsilon: float = -1.0
    pga: PgaParams = field(default_factory=PgaParams)

    def c(self):
        return _abi.rw_beta_params(self.beta_min, self.beta_max, self.epsilon, self.pga.c())


@dataclass
class BetaSearchResult:
    feasible: bool
    beta_star: Optional[float]
    w_star: Optional[RoutingFractions]
    best: RelaxedSolveResult
    trace: List[BetaStep]
    eval_passes: int = 0


@dataclass
class SetupSpace:
    models: List[str]
    tp_choices: List[List[int]]
    rho_choices: List[List[float]]

    def validate(self):  # setup_search.cpp:20-46
        if not self.models:
            raise ValidationError("setup space: no models")
        if len(set(self.models)) != len(self.models):
            dup = next(m for m in self.models if self.models.count(m) > 1)
            raise ValidationError(f"setup space: duplicate model '{dup}'")
        if len(self.tp_choices) != len(self.models) or len(self.rho_choices) != len(self.models):
            raise ValidationError("setup space: need tp and rho choices for every model")
        for i, name in enumerate(self.models):
            tps, rhos = self.tp_choices[i], self.rho_choices[i]
            if not tps or not rhos:
                raise ValidationError(f"setup space: model '{name}' has an empty choice set")
            for k, tp in enumerate(tps):
                if tp < 1:
                    raise ValidationError(f"setup space: model '{name}' tp choice must be >= 1")
                if k > 0 and tp <= tps[k - 1]:
                    raise ValidationError(
                        f"setup space: model '{name}' tp choices must be strictly increasing")
            for k, r in enumerate(rhos):
                if not (r > 0.0) or r > 1.0:
                    raise ValidationError(
                        f"setup space: model '{name}' rho choice must lie in (0, 1]")
                if k > 0 and r <= rhos[k - 1]:
                    raise ValidationError(
                        f"setup space: model '{name}' rho choices must be strictly increasing")


@dataclass
class SweepRecord:
    setup_id: int
    setup: SystemSetup
    score: float
    latency_ms: float
    feasible: bool


@dataclass
class PlanResult:
    feasible: bool = False
    setup: Optional[SystemSetup] = None
    w: Optional[RoutingFractions] = None
    beta: float = 0.0
    score: float = 0.0
    latency_ms: float = 0.0
    enumerated_count: int = 0
    retained_count: int = 0
    evaluated_count: int = 0
    per_model_load: List[float] = field(default_factory=list)
    out_of_range: List[bool] = field(default_factory=list)


@dataclass
class SearchContext:
    gpu_count: int = 1
    rho_floor: float = 1.0
    mem: Optional[MemoryTable] = None
    opt: OptimizeContext = field(default_factory=OptimizeContext)


@dataclass
class SearchParams:
    beta: BetaSearchParams = field(default_factory=BetaSearchParams)
    parallelism: int = 0  # GPUs are chosen by the caller's process layout; kept for parity


@dataclass
class SearchOutput:
    plan: PlanResult
    sweep: List[SweepRecord]
    records: Optional[np.ndarray] = None  # raw device records (RECORD_DTYPE)


class RetainVerdict(enum.IntEnum):
    RETAINED = 0
    UNDER_UTILIZED = 1
    OVER_BUDGET = 2
    PLACEMENT_INFEASIBLE = 3


# ---------------------------------------------------------------------------------------
# the GPU engine (one rw_ctx per device)


class Engine:
    """Owns one rw_ctx: the score matrix and profile table resident in HBM."""

    def __init__(self, device: int = 0):
        self.L = _abi.lib()
        h = C.c_void_p()
        rc = self.L.rw_create(device, C.byref(h))
        if rc:
            _raise(rc, self.L.rw_last_error(None).decode())
        self.h = h
        self.device = device
        self._scores_key = None
        self._profiles_key = None
        self.n = self.m = 0

    def close(self):
        if self.h:
            self.L.rw_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        if rc:
            _raise(rc, self.L.rw_last_error(self.h).decode())

    # inputs ---------------------------------------------------------------------------
    def set_stream(self, stream_handle: int):
        """Launch on this cudaStream_t.  0 selects the context's own stream (NOT the legacy
        default stream — pass 1, cudaStreamLegacy, for that); torch's default stream has
        handle 0, so share a torch.cuda.Stream() with the engine to order work."""
        self._chk(self.L.rw_set_stream(self.h, C.c_void_p(stream_handle)))

    def load_scores(self, scores: np.ndarray):
        a = np.ascontiguousarray(scores, dtype=np.float64)
        n, m = a.shape
        self._chk(self.L.rw_load_scores(self.h, n, m, dptr(a)))
        self.n, self.m = n, m
        self._scores_key = None
        return self

    def bind_scores_device(self, ptr: int, n: int, m: int):
        self._chk(self.L.rw_bind_scores_device(self.h, n, m, C.c_void_p(ptr)))
        self.n, self.m = n, m
        self._scores_key = None
        return self

    def ensure_scores(self, sm: ScoreMatrix):
        key = (id(sm), sm.scores.ctypes.data, sm.scores.shape)
        if self._scores_key != key:
            if sm.n() == 0 or sm.m() == 0:
                raise ValidationError("score matrix is empty")
            self.load_scores(sm.scores)
            self._scores_key = key

    def load_profiles(self, koff, kx, ky):
        koff = np.ascontiguousarray(koff, np.int64)
        kx = np.ascontiguousarray(kx, np.float64)
        ky = np.ascontiguousarray(ky, np.float64)
        self._chk(self.L.rw_load_profiles(self.h, len(koff) - 1, lptr(koff), dptr(kx), dptr(ky)))
        self._profiles_key = None
        return self

    def set_profiling(self, enable: bool = True):
        self._chk(self.L.rw_set_profiling(self.h, 1 if enable else 0))

    def profile(self) -> np.ndarray:
        out = np.zeros(32, np.int64)
        self._chk(self.L.rw_get_profile(self.h, lptr(out)))
        return out

    def last_kernel_ms(self) -> float:
        ms = C.c_double()
        self._chk(self.L.rw_last_kernel_ms(self.h, C.byref(ms)))
        return ms.value

    # solver entry points -------------------------------------------------------------
    def dual_objective(self, targets, alpha) -> float:
        t = np.ascontiguousarray(targets, np.float64)
        a = np.ascontiguousarray(alpha, np.float64)
        g = C.c_double()
        self._chk(self.L.rw_dual_objective(self.h, dptr(t), dptr(a), C.byref(g)))
        return g.value

    def assign_prompts(self, alpha):
        a = np.ascontiguousarray(alpha, np.float64)
        mo = np.zeros(self.n, np.int32)
        counts = np.zeros(max(self.m, 1), np.int32)
        self._chk(self.L.rw_assign_prompts(self.h, len(a), dptr(a), iptr(mo), iptr(counts)))
        return mo, counts[: self.m]

    def solve_dual(self, targets, params: SubgradientParams = SubgradientParams(),
                   init_alpha=None, want_assignment=True) -> DualSolution:
        t = np.ascontiguousarray(targets, np.float64)
        ia = None
        if init_alpha is not None and len(init_alpha) > 0:
            if len(init_alpha) != self.m:
                raise ValidationError("init_alpha has wrong length")
            ia = np.ascontiguousarray(init_alpha, np.float64)
        out = _abi.rw_dual_solution()
        asg = np.zeros(self.n, np.int32) if want_assignment else None
        p = params.c()
        self._chk(self.L.rw_solve_dual(self.h, dptr(t), C.byref(p), dptr(ia), C.byref(out),
                                       iptr(asg)))
        m = self.m
        return DualSolution(
            alpha_star=DualPrices(list(out.alpha_star[:m])), score=out.score,
            dual_bound=out.dual_bound, duality_gap=out.duality_gap,
            assignment=asg.tolist() if asg is not None else [],
            count_residual=list(out.count_residual[:m]), iterations=out.iterations,
            converged=bool(out.converged), counts=list(out.counts[:m]),
            eval_passes=out.eval_passes)

    def winner_policy(self, w_star, params: SubgradientParams = SubgradientParams(),
                      want_assignment=True):
        """The chosen setup's routing policy: cold solve_dual(N * w*) (test_cli.cpp:103-106)
        -> (DualSolution with counts, assignment as an int32 array)."""
        w = np.ascontiguousarray(w_star, np.float64)
        out = _abi.rw_dual_solution()
        asg = np.zeros(self.n, np.int32) if want_assignment else None
        p = params.c()
        self._chk(self.L.rw_winner_policy(self.h, len(w), dptr(w), C.byref(p), C.byref(out),
                                          iptr(asg)))
        m = self.m
        ds = DualSolution(
            alpha_star=DualPrices(list(out.alpha_star[:m])), score=out.score,
            dual_bound=out.dual_bound, duality_gap=out.duality_gap, assignment=[],
            count_residual=list(out.count_residual[:m]), iterations=out.iterations,
            converged=bool(out.converged), counts=list(out.counts[:m]),
            eval_passes=out.eval_passes)
        return ds, asg

    def project_simplex(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float64)
        w = np.zeros(max(len(v), 1))
        self._chk(self.L.rw_project_simplex(self.h, len(v), dptr(v), dptr(w)))
        return w[: len(v)]

    def system_latency_eval(self, profile_index, w, lambda_rps, kappa):
        pi = np.ascontiguousarray(profile_index, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        m = len(w)
        lat = C.c_double()
        loads, lats, grad = np.zeros(m), np.zeros(m), np.zeros(m)
        oor = np.zeros(m, np.int32)
        self._chk(self.L.rw_system_latency_eval(self.h, iptr(pi), dptr(w), lambda_rps, kappa,
                                                C.byref(lat), dptr(loads), dptr(lats),
                                                iptr(oor), dptr(grad)))
        return dict(latency=lat.value, loads=loads, lats=lats, oor=oor, grad=grad)

    def optimize_fractions(self, profile_index, beta, opt: OptimizeContext,
                           params: PgaParams = PgaParams()) -> RelaxedSolveResult:
        pi = np.ascontiguousarray(profile_index, np.int32)
        out = _abi.rw_relaxed_result()
        oc, pp = opt.c(), params.c()
        self._chk(self.L.rw_optimize_fractions(self.h, iptr(pi), beta, C.byref(oc), C.byref(pp),
                                               C.byref(out)))
        return _relaxed(out, self.m)

    def optimize_beta(self, profile_index, opt: OptimizeContext,
                      params: BetaSearchParams = BetaSearchParams(),
                      trace_cap: int = 128) -> BetaSearchResult:
        pi = np.ascontiguousarray(profile_index, np.int32)
        out = _abi.rw_beta_result()
        trace = (_abi.rw_beta_step * trace_cap)()
        oc, bp = opt.c(), params.c()
        self._chk(self.L.rw_optimize_beta(self.h, iptr(pi), C.byref(oc), C.byref(bp),
                                          C.byref(out), trace_cap, trace))
        m = self.m
        steps = [BetaStep(t.beta, t.score, t.latency_ms, bool(t.feasible))
                 for t in trace[: min(out.n_trace, trace_cap)]]
        feasible = bool(out.feasible)
        best = _relaxed(out.best, m) if feasible else RelaxedSolveResult(
            RoutingFractions([]), 0.0, 0.0, 0.0, 0, False, [])
        return BetaSearchResult(
            feasible=feasible, beta_star=out.beta_star if out.has_beta_star else None,
            w_star=RoutingFractions(list(out.w_star[:m])) if out.has_beta_star else None,
            best=best, trace=steps, eval_passes=out.eval_passes)

    def sweep(self, profile_index, setup_ids, opt: OptimizeContext,
              params: BetaSearchParams = BetaSearchParams(), shard_rank=0, shard_count=1):
        """Per-setup evaluate for this shard -> numpy array of RECORD_DTYPE."""
        pi = np.ascontiguousarray(profile_index, np.int32).reshape(-1)
        S = len(pi) // max(self.m, 1)
        ids = np.ascontiguousarray(setup_ids if setup_ids is not None else np.arange(S),
                                   np.int64)
        cap = max(1, (S - shard_rank + shard_count - 1) // shard_count)
        recs = np.zeros(cap, dtype=_abi.RECORD_DTYPE)
        n_out = C.c_int64()
        oc, bp = opt.c(), params.c()
        self._chk(self.L.rw_sweep(self.h, S, lptr(ids), iptr(pi), C.byref(oc), C.byref(bp),
                                  shard_rank, shard_count, C.c_void_p(recs.ctypes.data),
                                  C.byref(n_out)))
        return recs[: n_out.value]

    def sweep_slo(self, profile_index, setup_ids, taus, opt: OptimizeContext,
                  params: BetaSearchParams = BetaSearchParams(), shard_rank=0, shard_count=1):
        """All (setup, tau) instances in one launch -> records (tau-major instance order)."""
        self.sweep_async(profile_index, setup_ids, opt, params, shard_rank, shard_count, taus)
        return self.sweep_fetch()

    def sweep_async(self, profile_index, setup_ids, opt, params, shard_rank=0, shard_count=1,
                    taus=None):
        pi = np.ascontiguousarray(profile_index, np.int32).reshape(-1)
        S = len(pi) // max(self.m, 1)
        ids = np.ascontiguousarray(setup_ids if setup_ids is not None else np.arange(S),
                                   np.int64)
        t = np.ascontiguousarray([opt.tau_ms] if taus is None else taus, np.float64)
        plist = params if isinstance(params, (list, tuple)) else [params] * len(t)
        bps = (_abi.rw_beta_params * len(t))(*[q.c() for q in plist])
        self._pending = (pi, ids, t, S * len(t), shard_rank, shard_count)
        oc = opt.c()
        self._chk(self.L.rw_sweep_slo_async(self.h, S, lptr(ids), iptr(pi), len(t), dptr(t),
                                            C.byref(oc), bps, shard_rank, shard_count))

    def sweep_spec(self, profile_index, setup_ids, taus, opt: OptimizeContext, params,
                   depth: int = 2):
        """rw_sweep_spec: the sweep with a speculative beta bisection (depth levels/round)."""
        pi = np.ascontiguousarray(profile_index, np.int32).reshape(-1)
        S = len(pi) // max(self.m, 1)
        ids = np.ascontiguousarray(setup_ids if setup_ids is not None else np.arange(S),
                                   np.int64)
        t = np.ascontiguousarray(taus, np.float64)
        plist = params if isinstance(params, (list, tuple)) else [params] * len(t)
        bps = (_abi.rw_beta_params * len(t))(*[q.c() for q in plist])
        recs = np.zeros(max(S * len(t), 1), dtype=_abi.RECORD_DTYPE)
        n_out = C.c_int64()
        oc = opt.c()
        self._chk(self.L.rw_sweep_spec(self.h, S, lptr(ids), iptr(pi), len(t), dptr(t),
                                       C.byref(oc), bps, depth, C.c_void_p(recs.ctypes.data),
                                       C.byref(n_out)))
        return recs[: S * len(t)]

    def set_records_device(self, ptr: int, cap_records: int):
        """Sweeps write their records into this caller-owned device buffer (0 = ctx-owned)."""
        self._chk(self.L.rw_set_records_device(self.h, C.c_void_p(ptr or None),
                                               int(cap_records)))

    def sweep_fetch(self):
        _, _, _, S, r, cnt = self._pending
        cap = max(1, (S - r + cnt - 1) // cnt)
        recs = np.zeros(cap, dtype=_abi.RECORD_DTYPE)
        n_out = C.c_int64()
        self._chk(self.L.rw_sweep_fetch(self.h, C.c_void_p(recs.ctypes.data), C.byref(n_out)))
        return recs[: n_out.value]


def _relaxed(out, m) -> RelaxedSolveResult:
    return RelaxedSolveResult(
        w=RoutingFractions(list(out.w[:m])), objective=out.objective, score=out.score,
        latency_ms=out.latency_ms, iterations=out.iterations, converged=bool(out.converged),
        out_of_range=[bool((out.out_of_range >> i) & 1) for i in range(m)],
        eval_passes=out.eval_passes)


_ENGINES: Dict[int, Engine] = {}
_ENGINE_LOCK = threading.Lock()


def engine(device: int = 0) -> Engine:
    with _ENGINE_LOCK:
        if device not in _ENGINES:
            _ENGINES[device] = Engine(device)
        return _ENGINES[device]


def sweep_multi(engines: Sequence["Engine"], profile_index, setup_ids, taus,
                opt: OptimizeContext, params) -> np.ndarray:
    """rw_sweep_multi: the sweep sharded over several engines (one host thread per GPU);
    records in instance order, bit-identical to a one-engine sweep_slo."""
    pi = np.ascontiguousarray(profile_index, np.int32).reshape(-1)
    m = engines[0].m
    S = len(pi) // max(m, 1)
    ids = np.ascontiguousarray(setup_ids if setup_ids is not None else np.arange(S), np.int64)
    t = np.ascontiguousarray(taus, np.float64)
    plist = params if isinstance(params, (list, tuple)) else [params] * len(t)
    bps = (_abi.rw_beta_params * len(t))(*[q.c() for q in plist])
    hs = (C.c_void_p * len(engines))(*[e.h.value for e in engines])
    recs = np.zeros(max(S * len(t), 1), dtype=_abi.RECORD_DTYPE)
    oc = opt.c()
    rc = _abi.lib().rw_sweep_multi(hs, len(engines), S, lptr(ids), iptr(pi), len(t), dptr(t),
                                   C.byref(oc), bps, C.c_void_p(recs.ctypes.data))
    if rc:
        _raise(rc, _abi.lib().rw_last_error(engines[0].h).decode())
    return recs[: S * len(t)]


def reduce_records(records: np.ndarray) -> int:
    """setup_search.cpp:246-253 over records from any shards -> index or -1."""
    r = np.ascontiguousarray(records, dtype=_abi.RECORD_DTYPE)
    return int(_abi.lib().rw_reduce_records(len(r), C.c_void_p(r.ctypes.data)))


# ---------------------------------------------------------------------------------------
# reference-named free functions


def _check_dims(scores: ScoreMatrix, targets: TargetCounts):
    if scores.n() == 0 or scores.m() == 0:
        raise ValidationError("score matrix is empty")
    if targets.m() != scores.m():
        raise ValidationError(f"target counts have {targets.m()} entries for "
                              f"{scores.m()} models")


def assign_prompts(scores: ScoreMatrix, prices: DualPrices) -> Assignment:
    """score_dual.cpp:213-221."""
    e = engine()
    e.ensure_scores(scores)
    mo, counts = e.assign_prompts(prices.alpha)
    return Assignment(mo.tolist(), counts.tolist())


def dual_objective(scores: ScoreMatrix, targets: TargetCounts, prices: DualPrices) -> float:
    """score_dual.cpp:223-230."""
    _check_dims(scores, targets)
    if prices.m() != scores.m():
        raise ValidationError(f"prices have {prices.m()} entries for {scores.m()} models")
    e = engine()
    e.ensure_scores(scores)
    return e.dual_objective(targets.counts, prices.alpha)


def solve_dual(scores: ScoreMatrix, targets: TargetCounts,
               params: SubgradientParams = SubgradientParams()) -> DualSolution:
    """score_dual.cpp:232-327."""
    _check_dims(scores, targets)
    e = engine()
    e.ensure_scores(scores)
    return e.solve_dual(targets.counts, params, params.init_alpha or None)


def project_simplex(v: Sequence[float]) -> RoutingFractions:
    """routing_opt.cpp:37-68."""
    if len(v) == 0:
        raise ValidationError("project_simplex: empty input")
    if any(not math.isfinite(x) for x in v):
        raise ValidationError("project_simplex: non-finite input")
    return RoutingFractions(engine().project_simplex(v).tolist())


class _ProfileTableBuilder:
    """Resolves (model, tp, rho, metric) keys to rows of a device CSR profile table."""

    def __init__(self, lib: ProfileLibrary, metric: Metric):
        self.lib, self.metric = lib, metric
        self.index: Dict[tuple, int] = {}
        self.knots: List[List[Tuple[float, float]]] = []

    def idx(self, model, tp, rho) -> int:
        p = self.lib.at(model, tp, rho, self.metric)  # ConfigError naming the key
        key = (model, tp, quantize_rho(rho), int(self.metric))
        if key not in self.index:
            self.index[key] = len(self.knots)
            self.knots.append(list(p.knots))
        return self.index[key]

    def arrays(self):
        koff, kx, ky = [0], [], []
        for ks in self.knots:
            for x, y in ks:
                kx.append(float(x))
                ky.append(float(y))
            koff.append(len(kx))
        return (np.array(koff, np.int64), np.array(kx, np.float64), np.array(ky, np.float64))


def _check_context(setup: SystemSetup, ctx: OptimizeContext):
    """routing_opt.cpp:11-26."""
    if ctx.scores is None or ctx.lib is None:
        raise ValidationError("optimizer context: missing scores or profiles")
    setup.validate()
    if setup.m() != ctx.scores.m():
        raise ValidationError(f"setup has {setup.m()} models, score matrix has "
                              f"{ctx.scores.m()}")
    for i, ms in enumerate(setup.per_model):
        if ms.model != ctx.scores.models[i]:
            raise ValidationError(
                f"setup model order does not match score matrix (position {i}: "
                f"'{ms.model}' vs '{ctx.scores.models[i]}')")
    if not (ctx.lambda_rps > 0.0):
        raise ValidationError("arrival rate must be positive")
    if not (ctx.kappa > 0.0):
        raise ValidationError("kappa must be positive")
    b = _ProfileTableBuilder(ctx.lib, ctx.metric)
    pidx = [b.idx(ms.model, ms.tp, ms.rho) for ms in setup.per_model]
    e = engine()
    e.ensure_scores(ctx.scores)
    e.load_profiles(*b.arrays())
    return e, pidx


def system_latency_eval(lib: ProfileLibrary, setup: SystemSetup, w: RoutingFractions,
                        lambda_rps: float, metric: Metric, kappa: float):
    """latency.cpp:186-204 (+ grad, :429-441), evaluated on device."""
    if w.m() != setup.m():
        raise ValidationError(f"routing fractions have {w.m()} entries for {setup.m()} models")
    b = _ProfileTableBuilder(lib, metric)
    pidx = [b.idx(ms.model, ms.tp, ms.rho) for ms in setup.per_model]
    e = engine()
    if e.m != setup.m():  # latency needs an M-wide context; bind a dummy 1-row matrix
        e.load_scores(np.zeros((1, setup.m())))
        e._scores_key = None
    e.load_profiles(*b.arrays())
    return e.system_latency_eval(pidx, w.w, lambda_rps, kappa)


def optimize_fractions(setup: SystemSetup, beta: float, ctx: OptimizeContext,
                       params: PgaParams = PgaParams()) -> RelaxedSolveResult:
    """routing_opt.cpp:70-136."""
    e, pidx = _check_context(setup, ctx)
    if not (beta >= 0.0):
        raise ValidationError("beta must be >= 0")
    return e.optimize_fractions(pidx, beta, ctx, params)


def optimize_beta(setup: SystemSetup, ctx: OptimizeContext,
                  params: BetaSearchParams = BetaSearchParams()) -> BetaSearchResult:
    """routing_opt.cpp:138-173."""
    e, pidx = _check_context(setup, ctx)
    return e.optimize_beta(pidx, ctx, params)


def synth_scores(n_prompts: int, models: Sequence[str], shapes: Sequence[Tuple[float, float]],
                 seed: int) -> ScoreMatrix:
    """workload.cpp:78-112 (same mt19937_64 + libstdc++ gamma stream)."""
    if n_prompts < 1:
        raise ValidationError("synthetic workload: n_prompts must be >= 1")
    if not models:
        raise ValidationError("synthetic workload: no models")
    if len(shapes) != len(models):
        raise ValidationError("synthetic workload: need one (a, b) shape per model")
    for name, (a, b) in zip(models, shapes):
        if not (a > 0.0) or not (b > 0.0):
            raise ValidationError(f"synthetic workload: model '{name}' needs shape "
                                  "parameters a > 0 and b > 0")
    m = len(models)
    a = np.array([s[0] for s in shapes], np.float64)
    b = np.array([s[1] for s in shapes], np.float64)
    out = np.zeros((n_prompts, m), np.float64)
    rc = _abi.lib().rw_synth_scores(n_prompts, m, dptr(a), dptr(b), C.c_uint64(seed), dptr(out))
    if rc:
        _raise(rc, "synth_scores failed")
    return ScoreMatrix([f"p{j + 1}" for j in range(n_prompts)], list(models), out)


def write_scores_f64(matrix: ScoreMatrix, path: str) -> None:
    """f2: the score matrix as a RWSCORE1 binary file (rw_write_scores_f64)."""
    a = np.ascontiguousarray(matrix.scores, np.float64)
    n, m = a.shape
    names = (C.c_char_p * m)(*[s.encode() for s in matrix.models])
    rc = _abi.lib().rw_write_scores_f64(path.encode(), n, m, names, dptr(a))
    if rc:
        _raise(rc, _abi.lib().rw_host_last_error().decode())


def read_scores_f64(path: str) -> ScoreMatrix:
    """f2: a RWSCORE1 binary score file -> ScoreMatrix (validated like the CSV loader)."""
    L = _abi.lib()
    n, m = C.c_int64(), C.c_int32()
    names = C.create_string_buffer(1 << 16)
    rc = L.rw_read_scores_f64(path.encode(), C.byref(n), C.byref(m), None, 0, names, len(names))
    if rc:
        _raise(rc, L.rw_host_last_error().decode())
    out = np.empty((n.value, m.value), np.float64)
    rc = L.rw_read_scores_f64(path.encode(), None, None, dptr(out), out.size, None, 0)
    if rc:
        _raise(rc, L.rw_host_last_error().decode())
    models = names.raw.split(b"\0")[: m.value]
    return ScoreMatrix([f"p{j + 1}" for j in range(n.value)], [x.decode() for x in models], out)


def enumerate_retain(space: SetupSpace, gpu_count: int, rho_floor: float, mem: MemoryTable):
    """enumerate_setups + retain (setup_search.cpp:99-152) on the host C++ path.

    Returns (verdicts[E], tp[E, M], rho[E, M])."""
    space.validate()
    m = len(space.models)
    names = sorted(space.models, key=lambda s: s.encode())
    rank = np.array([names.index(x) for x in space.models], np.int32)
    tp_off = np.cumsum([0] + [len(t) for t in space.tp_choices]).astype(np.int32)
    tp_val = np.array([x for t in space.tp_choices for x in t], np.int32)
    rho_off = np.cumsum([0] + [len(r) for r in space.rho_choices]).astype(np.int32)
    rho_val = np.array([x for r in space.rho_choices for x in r], np.float64)
    ent = [(space.models.index(k[0]), k[1], v) for k, v in mem.entries.items()
           if k[0] in space.models]
    mm = np.array([e[0] for e in ent] or [0], np.int32)
    mt = np.array([e[1] for e in ent] or [0], np.int32)
    mf = np.array([e[2] for e in ent] or [0.0], np.float64)
    total = int(np.prod([len(t) * len(r) for t, r in zip(space.tp_choices, space.rho_choices)]))
    if gpu_count < 1:
        raise ValidationError("retain: GPU count must be >= 1")
    if not (rho_floor > 0.0) or rho_floor > 1.0:
        raise ValidationError("retain: rho_min must lie in (0, 1]")
    verdict = np.zeros(total, np.int32)
    tp_out = np.zeros((total, m), np.int32)
    rho_out = np.zeros((total, m), np.float64)
    n_enum = C.c_int64()
    rc = _abi.lib().rw_enumerate_retain(
        m, iptr(rank), iptr(tp_off), iptr(tp_val), iptr(rho_off), dptr(rho_val), len(ent),
        iptr(mm), iptr(mt), dptr(mf), gpu_count, rho_floor, total, C.byref(n_enum),
        iptr(verdict), iptr(tp_out), dptr(rho_out))
    if rc == _abi.RW_ERR_CONFIG:
        # name the first missing (model, tp) like MemoryTable::at (types.cpp:57-65)
        for i, name in enumerate(space.models):
            for tp in space.tp_choices[i]:
                mem.at(name, tp)
    if rc:
        _raise(rc, "enumerate/retain failed")
    return verdict, tp_out, rho_out


def select_setup(space: SetupSpace, ctx: SearchContext,
                 params: SearchParams = SearchParams(), *, shard_rank: int = 0,
                 shard_count: int = 1, gather: Optional[Callable] = None) -> SearchOutput:
    """setup_search.cpp:154-272 with the per-setup half on the GPU.

    Multi-GPU: each process passes its (shard_rank, shard_count) and a `gather` callable
    that all-gathers the fixed-size record array (e.g. torch.distributed over NCCL); the
    reduction is order-deterministic, so the result is identical for any GPU count.
    """
    space.validate()
    if ctx.mem is None:
        raise ValidationError("select_setup: missing memory table")
    if ctx.opt.scores is None or ctx.opt.lib is None:
        raise ValidationError("select_setup: missing scores or profiles")
    if list(ctx.opt.scores.models) != list(space.models):
        raise ValidationError("select_setup: score matrix columns must match the model list")
    verdict, tps, rhos = enumerate_retain(space, ctx.gpu_count, ctx.rho_floor, ctx.mem)
    retained = np.nonzero(verdict == 0)[0]
    beta_hi = params.beta.beta_max
    if beta_hi < 0.0:
        if not (ctx.opt.tau_ms > 0.0):
            raise ValidationError("latency target must be positive to derive default beta "
                                  "bounds")
    m = len(space.models)
    b = _ProfileTableBuilder(ctx.opt.lib, ctx.opt.metric)
    pidx = np.zeros((len(retained), m), np.int32)
    for r, k in enumerate(retained):
        for i in range(m):
            pidx[r, i] = b.idx(space.models[i], int(tps[k, i]), float(rhos[k, i]))
    if not (ctx.opt.lambda_rps > 0.0):
        raise ValidationError("arrival rate must be positive")
    if not (ctx.opt.kappa > 0.0):
        raise ValidationError("kappa must be positive")
    e = engine()
    e.ensure_scores(ctx.opt.scores)
    recs = np.zeros(0, dtype=_abi.RECORD_DTYPE)
    if len(retained):
        e.load_profiles(*b.arrays())
        recs = e.sweep(pidx, retained.astype(np.int64), ctx.opt, params.beta, shard_rank,
                       shard_count)
    if gather is not None:
        recs = gather(recs)
    recs = np.sort(recs, order="setup_id", kind="stable")

    def setup_of(k):
        return SystemSetup([ModelSetup(space.models[i], int(tps[k, i]), float(rhos[k, i]))
                            for i in range(m)])

    sweep = [SweepRecord(int(r["setup_id"]), setup_of(int(r["setup_id"])), float(r["score"]),
                         float(r["latency_ms"]), bool(r["feasible"])) for r in recs]
    plan = PlanResult(enumerated_count=len(verdict), retained_count=len(retained),
                      evaluated_count=len(retained))
    best = reduce_records(recs) if len(recs) else -1
    if best >= 0:
        r = recs[best]
        plan.feasible = True
        plan.setup = setup_of(int(r["setup_id"]))
        plan.w = RoutingFractions(list(r["w"][:m]))
        plan.beta = float(r["beta"])
        plan.score = float(r["score"])
        plan.latency_ms = float(r["latency_ms"])
        plan.out_of_range = [bool((int(r["out_of_range"]) >> i) & 1) for i in range(m)]
        plan.per_model_load = [ctx.opt.lambda_rps * x for x in plan.w.w]
    return SearchOutput(plan=plan, sweep=sweep, records=recs)
