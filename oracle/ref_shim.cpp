// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrappers over the UNMODIFIED reference library (routeplan, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  Tests use it
// to pin the C restatement (rw_oracle.c) and to generate golden fixtures; bench.py's
// reference arm times ref_select_setup on host cores.
//
// Flattened conventions shared with oracle/rw_oracle.h and include/rw_b200.h:
//   scores      row-major n*m doubles (workload.hpp:15 `scores[j * M + i]`)
//   profiles    CSR: koff[p+1], kx[], ky[] (latency.hpp:36 knots (load_rps, latency_ms))
//   status      0 ok, 1 ValidationError, 2 ConfigError, 9 other (errors.hpp:9-18)

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "routeplan/latency.hpp"
#include "routeplan/routing_opt.hpp"
#include "routeplan/score_dual.hpp"
#include "routeplan/setup_search.hpp"
#include "routeplan/types.hpp"
#include "routeplan/workload.hpp"

using namespace routeplan;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

std::string model_name(int i) { return "M" + std::to_string(i); }

ScoreMatrix make_matrix(int n, int m, const double* s) {
  ScoreMatrix sm;
  sm.prompts.reserve(n);
  for (int j = 0; j < n; ++j) sm.prompts.push_back("p" + std::to_string(j + 1));
  for (int i = 0; i < m; ++i) sm.models.push_back(model_name(i));
  sm.scores.assign(s, s + static_cast<size_t>(n) * m);
  return sm;
}

LatencyProfile make_profile(int i, int tp, double rho, const int64_t* koff, const double* kx,
                            const double* ky, int p) {
  LatencyProfile prof;
  prof.model = model_name(i);
  prof.tp = tp;
  prof.rho = rho;
  prof.metric = Metric::TTFT;
  for (int64_t k = koff[p]; k < koff[p + 1]; ++k) prof.knots.emplace_back(kx[k], ky[k]);
  return prof;
}

SubgradientParams sub_params(double eta0, int max_iters, double tol, int polish) {
  SubgradientParams p;
  p.eta0 = eta0;
  p.max_iters = max_iters;
  p.residual_tol = tol;
  p.polish_passes = polish;
  return p;
}

// One model-per-profile library for single-setup calls: model i uses profile i.
struct SingleSetup {
  ProfileLibrary lib;
  SystemSetup setup;
  SingleSetup(int m, const int64_t* koff, const double* kx, const double* ky) {
    for (int i = 0; i < m; ++i) {
      LatencyProfile p = make_profile(i, 1, 1.0, koff, kx, ky, i);
      lib.profiles[make_profile_key(p.model, 1, 1.0, Metric::TTFT)] = p;
      setup.per_model.push_back({model_name(i), 1, 1.0});
    }
  }
};

PgaParams pga_params(const double* pd, const int* pi) {
  // pd = {pga_eta, pga_w_tol, sub_eta0, sub_tol}; pi = {pga_max_iters, sub_max_iters, polish}
  PgaParams p;
  p.eta = pd[0];
  p.w_tol = pd[1];
  p.max_iters = pi[0];
  p.dual = sub_params(pd[2], pi[1], pd[3], pi[2]);
  return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_synth_scores(int n, int m, const double* a, const double* b, uint64_t seed, double* out) {
  return guarded([&] {
    std::vector<std::string> models;
    std::vector<BetaShape> shapes;
    for (int i = 0; i < m; ++i) {
      models.push_back(model_name(i));
      shapes.push_back({a[i], b[i]});
    }
    ScoreMatrix s = synth_scores(n, models, shapes, seed);
    std::memcpy(out, s.scores.data(), sizeof(double) * s.scores.size());
  });
}

int ref_dual_objective(int n, int m, const double* scores, const double* c, const double* alpha,
                       double* out_g) {
  return guarded([&] {
    ScoreMatrix s = make_matrix(n, m, scores);
    TargetCounts t;
    t.counts.assign(c, c + m);
    DualPrices p;
    p.alpha.assign(alpha, alpha + m);
    *out_g = dual_objective(s, t, p);
  });
}

int ref_assign_prompts(int n, int m, const double* scores, int m_alpha, const double* alpha,
                       int32_t* model_of, int32_t* counts) {
  return guarded([&] {
    ScoreMatrix s = make_matrix(n, m, scores);
    DualPrices p;
    p.alpha.assign(alpha, alpha + m_alpha);
    Assignment a = assign_prompts(s, p);
    for (int j = 0; j < n; ++j) model_of[j] = a.model_of[j];
    for (int i = 0; i < m; ++i) counts[i] = a.counts[i];
  });
}

// out_scalars = {score, dual_bound, duality_gap}; out_ints = {iterations, converged}
int ref_solve_dual(int n, int m, const double* scores, const double* c, double eta0,
                   int max_iters, double tol, int polish, const double* init_alpha,
                   double* alpha_star, double* out_scalars, int32_t* assignment,
                   double* residual, int32_t* out_ints) {
  return guarded([&] {
    ScoreMatrix s = make_matrix(n, m, scores);
    TargetCounts t;
    t.counts.assign(c, c + m);
    SubgradientParams p = sub_params(eta0, max_iters, tol, polish);
    if (init_alpha) p.init_alpha.assign(init_alpha, init_alpha + m);
    DualSolution d = solve_dual(s, t, p);
    for (int i = 0; i < m; ++i) {
      alpha_star[i] = d.alpha_star.alpha[i];
      residual[i] = d.count_residual[i];
    }
    out_scalars[0] = d.score;
    out_scalars[1] = d.dual_bound;
    out_scalars[2] = d.duality_gap;
    if (assignment)
      for (int j = 0; j < n; ++j) assignment[j] = d.assignment[j];
    out_ints[0] = d.iterations;
    out_ints[1] = d.converged ? 1 : 0;
  });
}

int ref_exact_score_oracle(int n, int m, const double* scores, const double* c, int max_n,
                           double* out) {
  return guarded([&] {
    ScoreMatrix s = make_matrix(n, m, scores);
    TargetCounts t;
    t.counts.assign(c, c + m);
    *out = exact_score_oracle(s, t, max_n);
  });
}

int ref_project_simplex(int m, const double* v, double* out) {
  return guarded([&] {
    RoutingFractions w = project_simplex(std::vector<double>(v, v + m));
    for (int i = 0; i < m; ++i) out[i] = w.w[i];
  });
}

int ref_latency_at(int nk, const double* kx, const double* ky, double load, double* out,
                   double* slope) {
  return guarded([&] {
    int64_t koff[2] = {0, nk};
    LatencyProfile p = make_profile(0, 1, 1.0, koff, kx, ky, 0);
    *out = latency_at(p, load);
    *slope = latency_slope(p, load);
  });
}

// out = {latency_ms}, per-model arrays load/lat/oor and grad.
int ref_system_latency_eval(int m, const int64_t* koff, const double* kx, const double* ky,
                            const double* w, double lambda, double kappa, double* latency,
                            double* loads, double* lats, int32_t* oor, double* grad) {
  return guarded([&] {
    SingleSetup ss(m, koff, kx, ky);
    RoutingFractions f;
    f.w.assign(w, w + m);
    SystemLatencyEval e = system_latency_eval(ss.lib, ss.setup, f, lambda, Metric::TTFT, kappa);
    *latency = e.latency_ms;
    std::vector<double> g = system_latency_grad(ss.lib, ss.setup, f, lambda, Metric::TTFT);
    for (int i = 0; i < m; ++i) {
      loads[i] = e.per_model_load[i];
      lats[i] = e.per_model_latency[i];
      oor[i] = e.out_of_range[i] ? 1 : 0;
      grad[i] = g[i];
    }
  });
}

// ctx = {lambda, tau, kappa}; pd/pi as pga_params.
// out_d = {objective, score, latency_ms}; out_i = {iterations, converged}
int ref_optimize_fractions(int n, int m, const double* scores, const int64_t* koff,
                           const double* kx, const double* ky, const double* ctx, double beta,
                           const double* pd, const int* pi, double* w_out, double* out_d,
                           int32_t* out_i, int32_t* oor) {
  return guarded([&] {
    ScoreMatrix s = make_matrix(n, m, scores);
    SingleSetup ss(m, koff, kx, ky);
    OptimizeContext oc;
    oc.scores = &s;
    oc.lib = &ss.lib;
    oc.lambda_rps = ctx[0];
    oc.tau_ms = ctx[1];
    oc.kappa = ctx[2];
    RelaxedSolveResult r = optimize_fractions(ss.setup, beta, oc, pga_params(pd, pi));
    for (int i = 0; i < m; ++i) {
      w_out[i] = r.w.w[i];
      oor[i] = r.out_of_range[i] ? 1 : 0;
    }
    out_d[0] = r.objective;
    out_d[1] = r.score;
    out_d[2] = r.latency_ms;
    out_i[0] = r.iterations;
    out_i[1] = r.converged ? 1 : 0;
  });
}

// bp = {beta_min, beta_max, epsilon}.
// out_d = {beta_star, best.objective, best.score, best.latency_ms}
// out_i = {feasible, has_beta_star, best.iterations, best.converged, n_trace}
// trace arrays sized trace_cap: beta, score, latency, feasible.
int ref_optimize_beta(int n, int m, const double* scores, const int64_t* koff, const double* kx,
                      const double* ky, const double* ctx, const double* bp, const double* pd,
                      const int* pi, double* w_star, double* best_w, int32_t* best_oor,
                      double* out_d, int32_t* out_i, int trace_cap, double* tr_beta,
                      double* tr_score, double* tr_lat, int32_t* tr_ok) {
  return guarded([&] {
    ScoreMatrix s = make_matrix(n, m, scores);
    SingleSetup ss(m, koff, kx, ky);
    OptimizeContext oc;
    oc.scores = &s;
    oc.lib = &ss.lib;
    oc.lambda_rps = ctx[0];
    oc.tau_ms = ctx[1];
    oc.kappa = ctx[2];
    BetaSearchParams b;
    b.beta_min = bp[0];
    b.beta_max = bp[1];
    b.epsilon = bp[2];
    b.pga = pga_params(pd, pi);
    BetaSearchResult r = optimize_beta(ss.setup, oc, b);
    out_i[0] = r.feasible ? 1 : 0;
    out_i[1] = r.beta_star.has_value() ? 1 : 0;
    out_d[0] = r.beta_star.value_or(0.0);
    out_d[1] = r.best.objective;
    out_d[2] = r.best.score;
    out_d[3] = r.best.latency_ms;
    out_i[2] = r.best.iterations;
    out_i[3] = r.best.converged ? 1 : 0;
    out_i[4] = static_cast<int32_t>(r.trace.size());
    for (int i = 0; i < m; ++i) {
      w_star[i] = r.w_star ? r.w_star->w[i] : 0.0;
      best_w[i] = r.best.w.w.empty() ? 0.0 : r.best.w.w[i];
      best_oor[i] = r.best.out_of_range.empty() ? 0 : (r.best.out_of_range[i] ? 1 : 0);
    }
    for (size_t k = 0; k < r.trace.size() && static_cast<int>(k) < trace_cap; ++k) {
      tr_beta[k] = r.trace[k].beta;
      tr_score[k] = r.trace[k].score;
      tr_lat[k] = r.trace[k].latency_ms;
      tr_ok[k] = r.trace[k].feasible ? 1 : 0;
    }
  });
}

// Full select_setup. Setup space: per model i, tp choices tp_vals[tp_off[i]..tp_off[i+1]),
// rho choices rho_vals[rho_off[i]..]. Memory table: n_mem entries (model, tp, frac).
// Profile table: n_prof entries (model, tp, rho) with CSR knots.
// sp = {gpu_count(as double), rho_floor, lambda, tau, kappa, beta_min, beta_max, epsilon,
//       pga_eta, pga_w_tol, sub_eta0, sub_tol}
// si = {pga_max_iters, sub_max_iters, polish, parallelism}
// outputs: counts = {enumerated, retained, plan_feasible}; sweep arrays sized sweep_cap;
// plan_d = {score, latency, beta}; plan_tp[m], plan_rho[m], plan_w[m], plan_load[m], plan_oor[m]
int ref_select_setup(int n, int m, const double* scores, const int* tp_off, const int* tp_vals,
                     const int* rho_off, const double* rho_vals, int n_mem, const int* mem_model,
                     const int* mem_tp, const double* mem_frac, int n_prof, const int* prof_model,
                     const int* prof_tp, const double* prof_rho, const int64_t* koff,
                     const double* kx, const double* ky, const double* sp, const int* si,
                     int64_t* counts, int sweep_cap, int64_t* sw_id, double* sw_score,
                     double* sw_lat, int32_t* sw_feas, double* plan_d, int32_t* plan_tp,
                     double* plan_rho, double* plan_w, double* plan_load, int32_t* plan_oor) {
  return guarded([&] {
    ScoreMatrix s = make_matrix(n, m, scores);
    SetupSpace space;
    for (int i = 0; i < m; ++i) {
      space.models.push_back(model_name(i));
      space.tp_choices.emplace_back(tp_vals + tp_off[i], tp_vals + tp_off[i + 1]);
      space.rho_choices.emplace_back(rho_vals + rho_off[i], rho_vals + rho_off[i + 1]);
    }
    MemoryTable mem;
    for (int k = 0; k < n_mem; ++k) mem.insert(model_name(mem_model[k]), mem_tp[k], mem_frac[k]);
    ProfileLibrary lib;
    for (int p = 0; p < n_prof; ++p) {
      LatencyProfile prof = make_profile(prof_model[p], prof_tp[p], prof_rho[p], koff, kx, ky, p);
      lib.profiles[make_profile_key(prof.model, prof.tp, prof.rho, Metric::TTFT)] = prof;
    }
    SearchContext ctx;
    ctx.gpu_count = static_cast<int>(sp[0]);
    ctx.rho_floor = sp[1];
    ctx.mem = &mem;
    ctx.opt.scores = &s;
    ctx.opt.lib = &lib;
    ctx.opt.lambda_rps = sp[2];
    ctx.opt.tau_ms = sp[3];
    ctx.opt.kappa = sp[4];
    SearchParams params;
    params.beta.beta_min = sp[5];
    params.beta.beta_max = sp[6];
    params.beta.epsilon = sp[7];
    params.beta.pga.eta = sp[8];
    params.beta.pga.w_tol = sp[9];
    params.beta.pga.max_iters = si[0];
    params.beta.pga.dual = sub_params(sp[10], si[1], sp[11], si[2]);
    params.parallelism = si[3];
    SearchOutput out = select_setup(space, ctx, params);
    counts[0] = out.plan.enumerated_count;
    counts[1] = out.plan.retained_count;
    counts[2] = out.plan.feasible ? 1 : 0;
    for (size_t k = 0; k < out.sweep.size() && static_cast<int>(k) < sweep_cap; ++k) {
      sw_id[k] = out.sweep[k].setup_id;
      sw_score[k] = out.sweep[k].score;
      sw_lat[k] = out.sweep[k].latency_ms;
      sw_feas[k] = out.sweep[k].feasible ? 1 : 0;
    }
    plan_d[0] = out.plan.score;
    plan_d[1] = out.plan.latency_ms;
    plan_d[2] = out.plan.beta;
    if (out.plan.feasible) {
      for (int i = 0; i < m; ++i) {
        plan_tp[i] = out.plan.setup.per_model[i].tp;
        plan_rho[i] = out.plan.setup.per_model[i].rho;
        plan_w[i] = out.plan.w.w[i];
        plan_load[i] = out.plan.per_model_load[i];
        plan_oor[i] = out.plan.out_of_range[i] ? 1 : 0;
      }
    }
  });
}

// Enumeration + retention only (setup_search.cpp:99-152). verdict per enumerated setup:
// 0 RETAINED, 1 UNDER_UTILIZED, 2 OVER_BUDGET, 3 PLACEMENT_INFEASIBLE.
int ref_enumerate_retain(int m, const int* tp_off, const int* tp_vals, const int* rho_off,
                         const double* rho_vals, int n_mem, const int* mem_model,
                         const int* mem_tp, const double* mem_frac, int gpu_count,
                         double rho_floor, int64_t cap, int64_t* n_enum, int32_t* verdict,
                         int32_t* tp_out, double* rho_out) {
  return guarded([&] {
    SetupSpace space;
    for (int i = 0; i < m; ++i) {
      space.models.push_back(model_name(i));
      space.tp_choices.emplace_back(tp_vals + tp_off[i], tp_vals + tp_off[i + 1]);
      space.rho_choices.emplace_back(rho_vals + rho_off[i], rho_vals + rho_off[i + 1]);
    }
    MemoryTable mem;
    for (int k = 0; k < n_mem; ++k) mem.insert(model_name(mem_model[k]), mem_tp[k], mem_frac[k]);
    std::vector<SystemSetup> all = enumerate_setups(space);
    *n_enum = static_cast<int64_t>(all.size());
    for (size_t k = 0; k < all.size() && static_cast<int64_t>(k) < cap; ++k) {
      verdict[k] = static_cast<int32_t>(retain(all[k], gpu_count, rho_floor, mem));
      for (int i = 0; i < m; ++i) {
        tp_out[k * m + i] = all[k].per_model[i].tp;
        rho_out[k * m + i] = all[k].per_model[i].rho;
      }
    }
  });
}

}  // extern "C"
