/* TEST INFRASTRUCTURE ONLY — see rw_oracle.h.  Each function cites the reference
 * file:line it restates.  Compiled with -ffp-contract=off (the reference build has no
 * FMA contraction). */
#include "rw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF (1.0 / 0.0)

/* std::max / std::min as libstdc++ defines them: max(a,b) = (a < b) ? b : a. */
static double smax(double a, double b) { return (a < b) ? b : a; }

/* ---- score_dual.cpp:25-49  eval_dual ------------------------------------------ */
double orc_eval_dual(int n, int m, const double* s, const double* c, const double* alpha,
                     int32_t* counts, int32_t* model_of, orc_counters* ctr) {
  if (ctr) ctr->eval_passes++;
  if (counts)
    for (int i = 0; i < m; ++i) counts[i] = 0;
  double sum = 0.0;
  for (int j = 0; j < n; ++j) {
    const double* row = s + (size_t)j * m;
    double best = row[0] - alpha[0];
    int arg = 0;
    for (int i = 1; i < m; ++i) {
      double v = row[i] - alpha[i];
      if (v > best) {
        best = v;
        arg = i;
      }
    }
    sum += best;
    if (counts) counts[arg]++;
    if (model_of) model_of[j] = arg;
  }
  for (int i = 0; i < m; ++i) sum += alpha[i] * c[i];
  return sum / n;
}

/* k-th largest value (1-based) of b[0..n): the value std::nth_element(greater) leaves
 * at position k-1 (score_dual.cpp:71-72).  Three-way quickselect; permutes b. */
static double kth_largest(double* b, int n, int k) {
  int lo = 0, hi = n; /* search window [lo, hi), target index k-1 in descending order */
  int target = k - 1;
  unsigned seed = 12345u;
  while (hi - lo > 1) {
    seed = seed * 1103515245u + 12345u;
    double pivot = b[lo + (int)(seed % (unsigned)(hi - lo))];
    /* partition into > pivot | == pivot | < pivot */
    int lt = lo, i = lo, gt = hi;
    while (i < gt) {
      if (b[i] > pivot) {
        double t = b[lt]; b[lt] = b[i]; b[i] = t;
        lt++; i++;
      } else if (b[i] < pivot) {
        gt--;
        double t = b[gt]; b[gt] = b[i]; b[i] = t;
      } else {
        i++;
      }
    }
    if (target < lt) hi = lt;
    else if (target >= gt) lo = gt;
    else return pivot;
  }
  return b[lo];
}

/* ---- score_dual.cpp:54-76  polish_pass ---------------------------------------- */
static void polish_pass(int n, int m, const double* s, const double* c, double* alpha,
                        double* b, double* max_delta, orc_counters* ctr) {
  if (ctr) ctr->polish_passes++;
  *max_delta = 0.0;
  for (int i = 0; i < m; ++i) {
    for (int j = 0; j < n; ++j) {
      const double* row = s + (size_t)j * m;
      double rest = -ORC_INF;
      for (int k = 0; k < m; ++k) {
        if (k == i) continue;
        rest = smax(rest, row[k] - alpha[k]);
      }
      b[j] = row[i] - rest;
    }
    int k = c[i] > 1e-12 ? (int)ceil(c[i] - 1e-9) : 1;
    if (k < 1) k = 1;
    if (k > n) k = n;
    double next = kth_largest(b, n, k);
    *max_delta = smax(*max_delta, fabs(next - alpha[i]));
    alpha[i] = next;
  }
}

/* ---- score_dual.cpp:81-185  repair_counts ------------------------------------- */
static double repair_counts(int n, int m, const double* s, const int32_t* target,
                            int32_t* model_of, int32_t* counts, orc_counters* ctr) {
  if (ctr) ctr->repair_calls++;
  int32_t delta[64];
  for (int i = 0; i < m; ++i) delta[i] = counts[i] - target[i];
#define MOVE(jj, vv)                 \
  do {                               \
    int u_ = model_of[(jj)];         \
    model_of[(jj)] = (vv);           \
    counts[u_]--; counts[(vv)]++;    \
    delta[u_]--; delta[(vv)]++;      \
  } while (0)
  /* Phase 1 (:96-118) */
  for (;;) {
    int over = 0;
    for (int i = 0; i < m; ++i) over = over || delta[i] > 0;
    if (!over) break;
    double best_loss = ORC_INF;
    int best_j = -1, best_v = -1;
    for (int j = 0; j < n; ++j) {
      int u = model_of[j];
      if (delta[u] <= 0) continue;
      const double* row = s + (size_t)j * m;
      for (int v = 0; v < m; ++v) {
        if (delta[v] >= 0) continue;
        double loss = row[u] - row[v];
        if (loss < best_loss) {
          best_loss = loss;
          best_j = j;
          best_v = v;
        }
      }
    }
    MOVE(best_j, best_v);
  }
  /* Phase 2 (:120-180) */
  if (m >= 2) {
    double* gain = (double*)malloc(sizeof(double) * m * m);
    int* witness = (int*)malloc(sizeof(int) * m * m);
    for (int pass = 0; pass < 10000; ++pass) {
      for (int q = 0; q < m * m; ++q) {
        gain[q] = -ORC_INF;
        witness[q] = -1;
      }
      for (int j = 0; j < n; ++j) {
        int u = model_of[j];
        const double* row = s + (size_t)j * m;
        for (int v = 0; v < m; ++v) {
          if (v == u) continue;
          double g = row[v] - row[u];
          if (g > gain[u * m + v]) {
            gain[u * m + v] = g;
            witness[u * m + v] = j;
          }
        }
      }
      double best = 1e-15;
      int cu = -1, cv = -1, cw = -1;
      for (int u = 0; u < m; ++u)
        for (int v = u + 1; v < m; ++v) {
          double g = gain[u * m + v] + gain[v * m + u];
          if (g > best) {
            best = g;
            cu = u; cv = v; cw = -1;
          }
        }
      for (int u = 0; u < m; ++u)
        for (int v = 0; v < m; ++v) {
          if (v == u) continue;
          for (int w = 0; w < m; ++w) {
            if (w == u || w == v) continue;
            double g = gain[u * m + v] + gain[v * m + w] + gain[w * m + u];
            if (g > best) {
              best = g;
              cu = u; cv = v; cw = w;
            }
          }
        }
      if (cu < 0) break;
      if (cw < 0) {
        int j1 = witness[cu * m + cv], j2 = witness[cv * m + cu];
        MOVE(j1, cv);
        MOVE(j2, cu);
      } else {
        int j1 = witness[cu * m + cv], j2 = witness[cv * m + cw], j3 = witness[cw * m + cu];
        MOVE(j1, cv);
        MOVE(j2, cw);
        MOVE(j3, cu);
      }
    }
    free(gain);
    free(witness);
  }
#undef MOVE
  double sum = 0.0;
  for (int j = 0; j < n; ++j) sum += s[(size_t)j * m + model_of[j]];
  return sum / n;
}

/* ---- score_dual.cpp:195-211  TargetCounts::validate / integral ----------------- */
static int targets_valid(int n, int m, const double* c) {
  if (m <= 0) return 0;
  double t = 0.0;
  for (int i = 0; i < m; ++i) {
    if (!isfinite(c[i]) || c[i] < -1e-9) return 0;
    t += c[i];
  }
  double scale = (double)n > 1.0 ? (double)n : 1.0;
  return fabs(t - n) <= 1e-6 * scale;
}

static int targets_integral(int m, const double* c) {
  for (int i = 0; i < m; ++i)
    if (fabs(c[i] - round(c[i])) > 1e-9) return 0;
  return 1;
}

/* ---- score_dual.cpp:232-327  solve_dual ---------------------------------------- */
int orc_solve_dual(int n, int m, const double* s, const double* c, const orc_sub_params* p,
                   const double* init_alpha, double* alpha_star, double* score,
                   double* dual_bound, double* gap, int32_t* assignment, double* residual,
                   int32_t* iterations, int32_t* converged, orc_counters* ctr) {
  if (n <= 0 || m <= 0 || m > 64) return 1;
  if (!targets_valid(n, m, c)) return 1;
  if (ctr) ctr->solves++;
  if (m == 1) { /* :239-249 */
    double sum = 0.0;
    for (int j = 0; j < n; ++j) sum += s[j];
    alpha_star[0] = 0.0;
    *score = *dual_bound = sum / n;
    *gap = 0.0;
    if (assignment)
      for (int j = 0; j < n; ++j) assignment[j] = 0;
    residual[0] = (n - c[0]) / n;
    *iterations = 0;
    *converged = 1;
    return 0;
  }
  double alpha[64], best_alpha[64], zero[64], polished[64];
  int32_t counts[64];
  for (int i = 0; i < m; ++i) {
    alpha[i] = init_alpha ? init_alpha[i] : 0.0;
    zero[i] = 0.0;
  }
  memcpy(best_alpha, alpha, sizeof(double) * m);
  double best_g = ORC_INF;
#define CONSIDER(a, g)                                   \
  do {                                                   \
    double g_ = (g);                                     \
    if (g_ < best_g) {                                   \
      best_g = g_;                                       \
      memcpy(best_alpha, (a), sizeof(double) * m);       \
    }                                                    \
  } while (0)
  CONSIDER(zero, orc_eval_dual(n, m, s, c, zero, NULL, NULL, ctr));
  *converged = 0;
  *iterations = 0;
  for (int t = 0; t < p->max_iters; ++t) {
    double g = orc_eval_dual(n, m, s, c, alpha, counts, NULL, ctr);
    CONSIDER(alpha, g);
    *iterations = t + 1;
    double resid = 0.0;
    for (int i = 0; i < m; ++i) resid = smax(resid, fabs(counts[i] - c[i]));
    resid /= n;
    if (resid <= p->residual_tol) {
      *converged = 1;
      break;
    }
    double eta = p->eta0 / sqrt((double)t + 1.0);
    for (int i = 0; i < m; ++i) alpha[i] += eta * (counts[i] - c[i]) / n;
  }
  /* :297-306 polish */
  memcpy(polished, best_alpha, sizeof(double) * m);
  double* b = (double*)malloc(sizeof(double) * (size_t)n);
  for (int pass = 0; pass < p->polish_passes; ++pass) {
    double max_delta = 0.0;
    polish_pass(n, m, s, c, polished, b, &max_delta, ctr);
    CONSIDER(polished, orc_eval_dual(n, m, s, c, polished, NULL, NULL, ctr));
    if (max_delta <= 1e-15) {
      *converged = 1;
      break;
    }
  }
  free(b);
#undef CONSIDER
  /* :309-310 gauge */
  double lo = best_alpha[0];
  for (int i = 1; i < m; ++i)
    if (best_alpha[i] < lo) lo = best_alpha[i];
  for (int i = 0; i < m; ++i) best_alpha[i] -= lo;
  memcpy(alpha_star, best_alpha, sizeof(double) * m);
  int32_t* asg = assignment ? assignment : (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  *dual_bound = orc_eval_dual(n, m, s, c, best_alpha, counts, asg, ctr);
  for (int i = 0; i < m; ++i) residual[i] = (counts[i] - c[i]) / n;
  if (targets_integral(m, c)) {
    int32_t target[64];
    for (int i = 0; i < m; ++i) target[i] = (int32_t)llround(c[i]);
    *score = repair_counts(n, m, s, target, asg, counts, ctr);
    *gap = *dual_bound - *score;
  } else {
    *score = *dual_bound;
    *gap = 0.0;
  }
  if (!assignment) free(asg);
  return 0;
}

/* ---- routing_opt.cpp:37-68  project_simplex ------------------------------------ */
int orc_project_simplex(int m, const double* v, double* w) {
  if (m <= 0) return 1;
  double u[64];
  for (int i = 0; i < m; ++i) {
    if (!isfinite(v[i])) return 1;
    u[i] = v[i];
  }
  for (int i = 1; i < m; ++i) { /* descending insertion sort (values only matter) */
    double x = u[i];
    int k = i - 1;
    while (k >= 0 && u[k] < x) {
      u[k + 1] = u[k];
      --k;
    }
    u[k + 1] = x;
  }
  double css = 0.0, theta = 0.0;
  for (int k = 0; k < m; ++k) {
    css += u[k];
    double t = (css - 1.0) / (k + 1);
    if (u[k] > t) theta = t;
  }
  double sum = 0.0;
  for (int i = 0; i < m; ++i) {
    w[i] = smax(v[i] - theta, 0.0);
    sum += w[i];
  }
  for (int i = 0; i < m; ++i) w[i] /= sum;
  return 0;
}

/* ---- latency.cpp:15-26, 140-157 ------------------------------------------------ */
static int64_t upper_knot(const orc_profiles* lib, int prof, double load) {
  int64_t a = lib->koff[prof], b = lib->koff[prof + 1];
  int64_t lo = a, hi = b; /* first k with load < kx[k] */
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (load < lib->kx[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo - a;
}

static double segment_slope(const orc_profiles* lib, int prof, int64_t hi) {
  int64_t base = lib->koff[prof];
  double x1 = lib->kx[base + hi - 1], y1 = lib->ky[base + hi - 1];
  double x2 = lib->kx[base + hi], y2 = lib->ky[base + hi];
  return (y2 - y1) / (x2 - x1);
}

double orc_latency_at(const orc_profiles* lib, int prof, double load) {
  int64_t nk = lib->koff[prof + 1] - lib->koff[prof];
  int64_t hi = upper_knot(lib, prof, load);
  int64_t base = lib->koff[prof];
  if (hi == 0) return lib->ky[base];
  if (hi == nk) hi = nk - 1;
  double x1 = lib->kx[base + hi - 1], y1 = lib->ky[base + hi - 1];
  return y1 + (load - x1) * segment_slope(lib, prof, hi);
}

double orc_latency_slope(const orc_profiles* lib, int prof, double load) {
  int64_t nk = lib->koff[prof + 1] - lib->koff[prof];
  int64_t hi = upper_knot(lib, prof, load);
  if (hi == 0) return 0.0;
  if (hi == nk) hi = nk - 1;
  return segment_slope(lib, prof, hi);
}

/* ---- latency.cpp:186-204  system_latency_eval --------------------------------- */
void orc_system_latency_eval(const orc_profiles* lib, const int32_t* prof_idx, int m,
                             const double* w, double lambda, double kappa, double* latency,
                             double* loads, double* lats, int32_t* oor) {
  double total = 0.0;
  for (int i = 0; i < m; ++i) {
    int p = prof_idx[i];
    double load = lambda * w[i];
    double lat = orc_latency_at(lib, p, load);
    double max_load = lib->kx[lib->koff[p + 1] - 1];
    if (loads) loads[i] = load;
    if (lats) lats[i] = lat;
    if (oor) oor[i] = load > kappa * max_load;
    if (w[i] != 0.0) total += w[i] * lat;
  }
  *latency = total;
}

/* ---- latency.cpp:172-184  system_latency_grad --------------------------------- */
void orc_system_latency_grad(const orc_profiles* lib, const int32_t* prof_idx, int m,
                             const double* w, double lambda, double* grad) {
  for (int i = 0; i < m; ++i) {
    double load = lambda * w[i];
    grad[i] = orc_latency_at(lib, prof_idx[i], load) +
              load * orc_latency_slope(lib, prof_idx[i], load);
  }
}

/* ---- routing_opt.cpp:70-136  optimize_fractions -------------------------------- */
int orc_optimize_fractions(int n, int m, const double* s, const orc_profiles* lib,
                           const int32_t* prof_idx, double beta, const orc_ctx* ctx,
                           const orc_pga_params* p, double* w_out, int32_t* oor_out,
                           orc_relaxed* out, orc_counters* ctr) {
  if (!(beta >= 0.0)) return 1;
  double w[64], best_w[64], warm[64], c[64], alpha[64], resid[64], grad[64], step[64],
      next[64];
  int have_warm = 0;
  for (int i = 0; i < m; ++i) w[i] = 1.0 / m;
  double best_obj = -ORC_INF;
  memcpy(best_w, w, sizeof(double) * m);
  int iterations = 0, converged = 0;
  for (int t = 0; t < p->max_iters; ++t) {
    for (int i = 0; i < m; ++i) c[i] = n * w[i];
    double sc, db, gp;
    int32_t it, cv;
    int rc = orc_solve_dual(n, m, s, c, &p->dual, have_warm ? warm : NULL, alpha, &sc, &db,
                            &gp, NULL, resid, &it, &cv, ctr);
    if (rc) return rc;
    memcpy(warm, alpha, sizeof(double) * m);
    have_warm = 1;
    double lat;
    orc_system_latency_eval(lib, prof_idx, m, w, ctx->lambda_rps, ctx->kappa, &lat, NULL, NULL,
                            NULL);
    double obj = db - beta * (lat - ctx->tau_ms);
    if (obj > best_obj) {
      best_obj = obj;
      memcpy(best_w, w, sizeof(double) * m);
    }
    iterations = t + 1;
    orc_system_latency_grad(lib, prof_idx, m, w, ctx->lambda_rps, grad);
    for (int i = 0; i < m; ++i) step[i] = w[i] + p->eta * (alpha[i] - beta * grad[i]);
    if (orc_project_simplex(m, step, next)) return 1;
    double moved = 0.0;
    for (int i = 0; i < m; ++i) moved = smax(moved, fabs(next[i] - w[i]));
    memcpy(w, next, sizeof(double) * m);
    if (moved <= p->w_tol) {
      converged = 1;
      break;
    }
  }
  for (int i = 0; i < m; ++i) c[i] = n * best_w[i];
  double sc, db, gp;
  int32_t it, cv;
  int rc = orc_solve_dual(n, m, s, c, &p->dual, NULL, alpha, &sc, &db, &gp, NULL, resid, &it,
                          &cv, ctr);
  if (rc) return rc;
  double lat;
  orc_system_latency_eval(lib, prof_idx, m, best_w, ctx->lambda_rps, ctx->kappa, &lat, NULL,
                          NULL, oor_out);
  memcpy(w_out, best_w, sizeof(double) * m);
  out->score = sc;
  out->latency_ms = lat;
  out->objective = sc - beta * (lat - ctx->tau_ms);
  out->iterations = iterations;
  out->converged = converged;
  return 0;
}

/* ---- routing_opt.cpp:138-173  optimize_beta ------------------------------------ */
int orc_optimize_beta(int n, int m, const double* s, const orc_profiles* lib,
                      const int32_t* prof_idx, const orc_ctx* ctx, const orc_beta_params* p,
                      double* w_star, double* best_w, int32_t* best_oor, orc_beta_result* out,
                      int trace_cap, double* tr_beta, double* tr_score, double* tr_lat,
                      int32_t* tr_ok, orc_counters* ctr) {
  double lo = p->beta_min, hi = p->beta_max;
  if (hi < 0.0) {
    if (!(ctx->tau_ms > 0.0)) return 1;
    hi = 10.0 / ctx->tau_ms;
  }
  double eps = p->epsilon;
  if (eps < 0.0) eps = (hi - lo) / 1024.0;
  if (!(lo >= 0.0) || !(lo < hi)) return 1;
  if (!(eps > 0.0)) return 1;
  memset(out, 0, sizeof(*out));
  double w[64];
  int32_t oor[64];
  while (hi - lo > eps) {
    double mid = 0.5 * (lo + hi);
    orc_relaxed r;
    int rc = orc_optimize_fractions(n, m, s, lib, prof_idx, mid, ctx, &p->pga, w, oor, &r, ctr);
    if (rc) return rc;
    int in_range = 1;
    for (int i = 0; i < m; ++i)
      if (oor[i]) in_range = 0;
    int ok = r.latency_ms <= ctx->tau_ms && in_range;
    if (out->n_trace < trace_cap) {
      tr_beta[out->n_trace] = mid;
      tr_score[out->n_trace] = r.score;
      tr_lat[out->n_trace] = r.latency_ms;
      tr_ok[out->n_trace] = ok;
    }
    out->n_trace++;
    if (ok) {
      out->feasible = 1;
      out->has_beta_star = 1;
      out->beta_star = mid;
      memcpy(w_star, w, sizeof(double) * m);
      memcpy(best_w, w, sizeof(double) * m);
      memcpy(best_oor, oor, sizeof(int32_t) * m);
      out->best = r;
      hi = mid;
    } else {
      lo = mid;
    }
  }
  return 0;
}

/* ---- setup_search.cpp:187-211  evaluate ---------------------------------------- */
int orc_evaluate_setup(int n, int m, const double* s, const orc_profiles* lib,
                       const int32_t* prof_idx, const orc_ctx* ctx, const orc_beta_params* p,
                       orc_setup_eval* out, double* w_out, int32_t* oor_out, orc_counters* ctr) {
  enum { CAP = 256 };
  double tr_beta[CAP], tr_score[CAP], tr_lat[CAP], w_star[64], best_w[64];
  int32_t tr_ok[CAP], best_oor[64];
  orc_beta_result br;
  int rc = orc_optimize_beta(n, m, s, lib, prof_idx, ctx, p, w_star, best_w, best_oor, &br, CAP,
                             tr_beta, tr_score, tr_lat, tr_ok, ctr);
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  for (int i = 0; i < m; ++i) {
    w_out[i] = 0.0;
    oor_out[i] = 0;
  }
  if (br.feasible) {
    out->feasible = 1;
    out->score = br.best.score;
    out->latency_ms = br.best.latency_ms;
    out->beta = br.beta_star;
    memcpy(w_out, best_w, sizeof(double) * m);
    memcpy(oor_out, best_oor, sizeof(int32_t) * m);
  } else if (br.n_trace > 0) {
    int nt = br.n_trace < CAP ? br.n_trace : CAP;
    int best = 0;
    for (int k = 1; k < nt; ++k)
      if (tr_lat[k] < tr_lat[best]) best = k;
    out->score = tr_score[best];
    out->latency_ms = tr_lat[best];
  } else {
    double beta_hi = p->beta_max;
    if (beta_hi < 0.0) beta_hi = 10.0 / ctx->tau_ms;
    orc_relaxed r;
    double w[64];
    int32_t oor[64];
    rc = orc_optimize_fractions(n, m, s, lib, prof_idx, beta_hi, ctx, &p->pga, w, oor, &r, ctr);
    if (rc) return rc;
    out->score = r.score;
    out->latency_ms = r.latency_ms;
  }
  return 0;
}

/* ---- setup_search.cpp:246-253  reduction ---------------------------------------- */
int64_t orc_reduce(int64_t count, const int32_t* feasible, const double* score,
                   const double* latency) {
  int64_t best = -1;
  for (int64_t k = 0; k < count; ++k) {
    if (!feasible[k]) continue;
    if (best < 0 || score[k] > score[best] ||
        (score[k] == score[best] && latency[k] < latency[best]))
      best = k;
  }
  return best;
}
