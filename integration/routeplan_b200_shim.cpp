// routeplan_b200_shim.cpp — the reference-side binding of the B200 path.
//
// Link-time drop-in for the reference C++ library (/root/reference/proj): this file
// defines the hot-path entry points of `routeplan` over the C-ABI of include/rw_b200.h,
// so the reference's own callers (runner.cpp `run_search`, the doctest suite, the
// acceptance binary) run on the GPU unchanged.  The reference definitions of the same
// functions are compiled out of their translation units by renaming (see Makefile here:
// -Dsolve_dual=ref_cpu_solve_dual on score_dual.cpp, ...); nothing else changes.
//
// Replaced entry points (reference declaration -> C-ABI call):
//   score_dual.hpp:34  assign_prompts      -> rw_assign_prompts
//   score_dual.hpp:38  dual_objective      -> rw_dual_objective
//   score_dual.hpp:64  solve_dual          -> rw_solve_dual
//   routing_opt.hpp:50 optimize_fractions  -> rw_optimize_fractions
//   routing_opt.hpp:79 optimize_beta       -> rw_optimize_beta
//   setup_search.hpp:88 select_setup       -> rw_sweep (+ host enumerate/retain, reduction)
// Validation runs first with the reference's own validators and messages, so error
// behaviour (ValidationError / ConfigError, errors.hpp:9-18) is the reference's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "routeplan/errors.hpp"
#include "routeplan/latency.hpp"
#include "routeplan/routing_opt.hpp"
#include "routeplan/score_dual.hpp"
#include "routeplan/setup_search.hpp"
#include "rw_b200.h"

namespace routeplan {
namespace {

std::mutex g_mu;  // the reference functions are re-entrant; the shim serialises one ctx

rw_ctx* dev() {
  static rw_ctx* ctx = [] {
    rw_ctx* c = nullptr;
    if (rw_create(0, &c) != RW_OK)
      throw std::runtime_error(std::string("rw_create: ") + rw_last_error(nullptr));
    return c;
  }();
  return ctx;
}

// Contexts of shards 1.. of a multi-GPU select_setup: shard r lives on device r % #GPUs.
// (RW_SHIM_SHARED_GPU=1 lets more shards than GPUs share devices — a test hook that runs
// the multi-shard path on one GPU.)
rw_ctx* shard_ctx(int r) {
  static std::vector<rw_ctx*> ctxs;
  if (r == 0) return dev();
  while (static_cast<int>(ctxs.size()) < r) ctxs.push_back(nullptr);
  rw_ctx*& c = ctxs[r - 1];
  if (!c) {
    const int ndev = std::max(1, rw_device_count());
    if (rw_create(r % ndev, &c) != RW_OK)
      throw std::runtime_error(std::string("rw_create: ") + rw_last_error(nullptr));
  }
  return c;
}

void check(int rc) {
  if (rc == RW_OK) return;
  const std::string msg = rw_last_error(dev());
  if (rc == RW_ERR_VALIDATION || rc == RW_ERR_UNSUPPORTED) throw ValidationError(msg);
  if (rc == RW_ERR_CONFIG) throw ConfigError(msg);
  throw std::runtime_error("rw_b200: " + msg);
}

void upload(const ScoreMatrix& s, rw_ctx* c = nullptr) {
  check(rw_load_scores(c ? c : dev(), s.n(), s.m(), s.scores.data()));
}

void check_dims(const ScoreMatrix& scores, const TargetCounts& targets) {  // score_dual.cpp:15
  if (scores.prompts.empty() || scores.models.empty())
    throw ValidationError("score matrix is empty");
  if (targets.m() != scores.m())
    throw ValidationError("target counts have " + std::to_string(targets.m()) +
                          " entries for " + std::to_string(scores.m()) + " models");
  targets.validate(scores.n());
}

void check_context(const SystemSetup& setup, const OptimizeContext& ctx) {  // routing_opt.cpp:11
  if (!ctx.scores || !ctx.lib) throw ValidationError("optimizer context: missing scores or profiles");
  setup.validate();
  if (setup.m() != ctx.scores->m())
    throw ValidationError("setup has " + std::to_string(setup.m()) + " models, score matrix has " +
                          std::to_string(ctx.scores->m()));
  for (int i = 0; i < setup.m(); ++i)
    if (setup.per_model[i].model != ctx.scores->models[i])
      throw ValidationError("setup model order does not match score matrix (position " +
                            std::to_string(i) + ": '" + setup.per_model[i].model + "' vs '" +
                            ctx.scores->models[i] + "')");
  if (!(ctx.lambda_rps > 0.0)) throw ValidationError("arrival rate must be positive");
  if (!(ctx.kappa > 0.0)) throw ValidationError("kappa must be positive");
  for (const auto& ms : setup.per_model) ctx.lib->at(ms.model, ms.tp, ms.rho, ctx.metric);
}

// The CSR profile table of the (model, tp, rho, metric) keys the setups use, in
// first-use order; profile_index[k * M + i] names setup k's profile for model i.
struct ProfileTable {
  std::vector<int64_t> koff{0};
  std::vector<double> kx, ky;
  std::vector<int32_t> index;
  std::map<const LatencyProfile*, int32_t> seen;
  void add_setup(const SystemSetup& setup, const ProfileLibrary& lib, Metric metric) {
    for (const auto& ms : setup.per_model) {
      const LatencyProfile& p = lib.at(ms.model, ms.tp, ms.rho, metric);  // ConfigError
      auto it = seen.find(&p);
      if (it == seen.end()) {
        it = seen.emplace(&p, static_cast<int32_t>(koff.size() - 1)).first;
        for (const auto& [x, y] : p.knots) {
          kx.push_back(x);
          ky.push_back(y);
        }
        koff.push_back(static_cast<int64_t>(kx.size()));
      }
      index.push_back(it->second);
    }
  }
  void upload(rw_ctx* c = nullptr) const {
    check(rw_load_profiles(c ? c : dev(), static_cast<int32_t>(koff.size() - 1), koff.data(),
                           kx.data(), ky.data()));
  }
};

rw_subgradient_params sub_params(const SubgradientParams& p) {
  return rw_subgradient_params{p.eta0, p.max_iters, p.residual_tol, p.polish_passes};
}
rw_pga_params pga_params(const PgaParams& p) {
  if (p.on_iterate)  // per-iterate host callbacks would need a host round trip per iterate
    throw ValidationError("PgaParams::on_iterate is not supported by the B200 path");
  return rw_pga_params{p.eta, p.max_iters, p.w_tol, sub_params(p.dual)};
}
rw_beta_params beta_params(const BetaSearchParams& p) {
  return rw_beta_params{p.beta_min, p.beta_max, p.epsilon, pga_params(p.pga)};
}

RelaxedSolveResult relaxed(const rw_relaxed_result& r, int m) {
  RelaxedSolveResult out;
  out.w.w.assign(r.w, r.w + m);
  out.objective = r.objective;
  out.score = r.score;
  out.latency_ms = r.latency_ms;
  out.iterations = r.iterations;
  out.converged = r.converged != 0;
  out.out_of_range.resize(m);
  for (int i = 0; i < m; ++i) out.out_of_range[i] = (r.out_of_range >> i) & 1u;
  return out;
}

}  // namespace

Assignment assign_prompts(const ScoreMatrix& scores, const DualPrices& prices) {
  if (prices.m() != scores.m())  // score_dual.cpp:214-216
    throw ValidationError("prices have " + std::to_string(prices.m()) + " entries for " +
                          std::to_string(scores.m()) + " models");
  std::lock_guard<std::mutex> lk(g_mu);
  upload(scores);
  Assignment out;
  out.model_of.resize(scores.n());
  out.counts.resize(scores.m());
  std::vector<int32_t> mo(scores.n()), counts(scores.m());
  check(rw_assign_prompts(dev(), prices.m(), prices.alpha.data(), mo.data(), counts.data()));
  out.model_of.assign(mo.begin(), mo.end());
  out.counts.assign(counts.begin(), counts.end());
  return out;
}

double dual_objective(const ScoreMatrix& scores, const TargetCounts& targets,
                      const DualPrices& prices) {
  check_dims(scores, targets);
  if (prices.m() != scores.m())
    throw ValidationError("prices have " + std::to_string(prices.m()) + " entries for " +
                          std::to_string(scores.m()) + " models");
  std::lock_guard<std::mutex> lk(g_mu);
  upload(scores);
  double g = 0.0;
  check(rw_dual_objective(dev(), targets.counts.data(), prices.alpha.data(), &g));
  return g;
}

DualSolution solve_dual(const ScoreMatrix& scores, const TargetCounts& targets,
                        const SubgradientParams& params) {
  check_dims(scores, targets);
  const int n = scores.n(), m = scores.m();
  if (m > 1 && !params.init_alpha.empty() && static_cast<int>(params.init_alpha.size()) != m)
    throw ValidationError("init_alpha has wrong length");
  std::lock_guard<std::mutex> lk(g_mu);
  upload(scores);
  rw_subgradient_params p = sub_params(params);
  rw_dual_solution d;
  std::vector<int32_t> asg(n);
  check(rw_solve_dual(dev(), targets.counts.data(), &p,
                      (m > 1 && !params.init_alpha.empty()) ? params.init_alpha.data() : nullptr,
                      &d, asg.data()));
  DualSolution out;
  out.alpha_star.alpha.assign(d.alpha_star, d.alpha_star + m);
  out.score = d.score;
  out.dual_bound = d.dual_bound;
  out.duality_gap = d.duality_gap;
  out.assignment.assign(asg.begin(), asg.end());
  out.count_residual.assign(d.count_residual, d.count_residual + m);
  out.iterations = d.iterations;
  out.converged = d.converged != 0;
  return out;
}

RelaxedSolveResult optimize_fractions(const SystemSetup& setup, double beta,
                                      const OptimizeContext& ctx, const PgaParams& params) {
  check_context(setup, ctx);
  if (!(beta >= 0.0)) throw ValidationError("beta must be >= 0");
  ProfileTable t;
  t.add_setup(setup, *ctx.lib, ctx.metric);
  rw_pga_params p = pga_params(params);
  rw_opt_context oc{ctx.lambda_rps, ctx.tau_ms, ctx.kappa};
  std::lock_guard<std::mutex> lk(g_mu);
  upload(*ctx.scores);
  t.upload();
  rw_relaxed_result r;
  check(rw_optimize_fractions(dev(), t.index.data(), beta, &oc, &p, &r));
  return relaxed(r, setup.m());
}

BetaSearchResult optimize_beta(const SystemSetup& setup, const OptimizeContext& ctx,
                               const BetaSearchParams& params) {
  check_context(setup, ctx);
  ProfileTable t;
  t.add_setup(setup, *ctx.lib, ctx.metric);
  rw_beta_params p = beta_params(params);
  rw_opt_context oc{ctx.lambda_rps, ctx.tau_ms, ctx.kappa};
  std::lock_guard<std::mutex> lk(g_mu);
  upload(*ctx.scores);
  t.upload();
  rw_beta_result r;
  // every bisection step is returned, as the reference's trace holds them all: size the
  // buffer from the bracket (the span halves each step, routing_opt.cpp:154-171)
  double lo = params.beta_min, hi = params.beta_max;
  if (hi < 0.0 && ctx.tau_ms > 0.0) hi = 10.0 / ctx.tau_ms;
  double eps = params.epsilon < 0.0 ? (hi - lo) / 1024.0 : params.epsilon;
  int cap = RW_MAX_TRACE;
  if (hi > lo && eps > 0.0)
    cap = std::max(cap, static_cast<int>(std::ceil(std::log2((hi - lo) / eps))) + 8);
  std::vector<rw_beta_step> trace(cap);
  check(rw_optimize_beta(dev(), t.index.data(), &oc, &p, &r, cap, trace.data()));
  const int m = setup.m();
  BetaSearchResult out;
  out.feasible = r.feasible != 0;
  if (r.has_beta_star) {
    out.beta_star = r.beta_star;
    RoutingFractions w;
    w.w.assign(r.w_star, r.w_star + m);
    out.w_star = w;
  }
  if (out.feasible) out.best = relaxed(r.best, m);
  for (int k = 0; k < r.n_trace && k < cap; ++k)
    out.trace.push_back({trace[k].beta, trace[k].score, trace[k].latency_ms,
                         trace[k].feasible != 0});
  return out;
}

SearchOutput select_setup(const SetupSpace& space, const SearchContext& ctx,
                          const SearchParams& params) {
  // setup_search.cpp:154-166: validation, enumeration and retention on the host
  space.validate();
  if (!ctx.mem) throw ValidationError("select_setup: missing memory table");
  if (!ctx.opt.scores || !ctx.opt.lib)
    throw ValidationError("select_setup: missing scores or profiles");
  if (ctx.opt.scores->models != space.models)
    throw ValidationError("select_setup: score matrix columns must match the model list");
  std::vector<SystemSetup> all = enumerate_setups(space);
  std::vector<int64_t> retained_ids;
  for (size_t id = 0; id < all.size(); ++id)
    if (retain(all[id], ctx.gpu_count, ctx.rho_floor, *ctx.mem) == RetainVerdict::RETAINED)
      retained_ids.push_back(static_cast<int64_t>(id));
  double beta_hi = params.beta.beta_max;  // :169-174
  if (beta_hi < 0.0 && !(ctx.opt.tau_ms > 0.0))
    throw ValidationError("latency target must be positive to derive default beta bounds");

  SearchOutput out;
  PlanResult& plan = out.plan;
  plan.enumerated_count = static_cast<long>(all.size());
  plan.retained_count = static_cast<long>(retained_ids.size());
  plan.evaluated_count = static_cast<long>(retained_ids.size());
  if (retained_ids.empty()) return out;
  for (int64_t id : retained_ids) check_context(all[id], ctx.opt);

  // the per-setup half on the GPU: one persistent kernel over every retained setup
  ProfileTable t;
  for (int64_t id : retained_ids) t.add_setup(all[id], *ctx.opt.lib, ctx.opt.metric);
  rw_beta_params p = beta_params(params.beta);
  rw_opt_context oc{ctx.opt.lambda_rps, ctx.opt.tau_ms, ctx.opt.kappa};
  std::vector<rw_setup_record> recs(retained_ids.size());
  int64_t n_out = static_cast<int64_t>(retained_ids.size());
  // SearchParams::parallelism (setup_search.cpp:213-215: worker threads, <= 0 -> all) maps
  // to GPUs: shard r of W on GPU r, one host thread each, records gathered in setup order
  const int ndev = std::max(1, rw_device_count());
  const char* shared = std::getenv("RW_SHIM_SHARED_GPU");
  int shards = params.parallelism > 0 ? params.parallelism : ndev;
  if (!(shared && shared[0] == '1')) shards = std::min(shards, ndev);
  shards = std::clamp<int>(shards, 1, static_cast<int>(retained_ids.size()));
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (shards == 1) {
      upload(*ctx.opt.scores);
      t.upload();
      check(rw_sweep(dev(), static_cast<int64_t>(retained_ids.size()), retained_ids.data(),
                     t.index.data(), &oc, &p, 0, 1, recs.data(), &n_out));
    } else {
      std::vector<rw_ctx*> cs(shards);
      for (int r = 0; r < shards; ++r) {
        cs[r] = shard_ctx(r);
        upload(*ctx.opt.scores, cs[r]);
        t.upload(cs[r]);
      }
      const double tau = oc.tau_ms;
      check(rw_sweep_multi(cs.data(), shards, static_cast<int64_t>(retained_ids.size()),
                           retained_ids.data(), t.index.data(), 1, &tau, &oc, &p, recs.data()));
    }
  }
  out.sweep.reserve(retained_ids.size());
  for (size_t k = 0; k < retained_ids.size(); ++k)  // records come back in enumeration order
    out.sweep.push_back({static_cast<long>(recs[k].setup_id), all[retained_ids[k]],
                         recs[k].score, recs[k].latency_ms, recs[k].feasible != 0});
  const int64_t best = rw_reduce_records(n_out, recs.data());  // :246-253
  if (best >= 0) {
    const rw_setup_record& r = recs[best];
    const int m = static_cast<int>(space.models.size());
    plan.feasible = true;
    plan.setup = all[retained_ids[best]];
    plan.w.w.assign(r.w, r.w + m);
    plan.beta = r.beta;
    plan.score = r.score;
    plan.latency_ms = r.latency_ms;
    plan.out_of_range.resize(m);
    for (int i = 0; i < m; ++i) plan.out_of_range[i] = (r.out_of_range >> i) & 1u;
    plan.per_model_load.resize(m);
    for (int i = 0; i < m; ++i) plan.per_model_load[i] = ctx.opt.lambda_rps * plan.w.w[i];
  }
  return out;
}

}  // namespace routeplan
