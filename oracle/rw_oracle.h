/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of the RouterWise setup-search inner loop
 * (/root/reference/proj/src/{score_dual,latency,routing_opt,setup_search}.cpp).
 * Parity pinned against the compiled reference (oracle/_ref, tests/test_oracle_pin.py)
 * and against golden vectors in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg may
 * load this library.
 */
#ifndef RW_ORACLE_H
#define RW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double eta0;         /* score_dual.hpp:47 */
  int32_t max_iters;   /* :48 */
  double residual_tol; /* :49 */
  int32_t polish_passes; /* :50 */
} orc_sub_params;

typedef struct {
  double eta;        /* routing_opt.hpp:28 */
  int32_t max_iters; /* :29 */
  double w_tol;      /* :30 */
  orc_sub_params dual;
} orc_pga_params;

typedef struct {
  double beta_min, beta_max, epsilon; /* routing_opt.hpp:70-72 */
  orc_pga_params pga;
} orc_beta_params;

typedef struct {
  double lambda_rps, tau_ms, kappa; /* routing_opt.hpp:21-24 */
} orc_ctx;

/* Instrumentation (counts only, no arithmetic effect). */
typedef struct {
  int64_t eval_passes;   /* eval_dual calls (the "evals" unit) */
  int64_t polish_passes; /* polish_pass calls */
  int64_t repair_calls;  /* repair_counts calls */
  int64_t solves;        /* solve_dual calls */
} orc_counters;

/* Latency profile table in CSR form: profile p has knots [koff[p], koff[p+1]). */
typedef struct {
  const int64_t* koff;
  const double* kx; /* load_rps */
  const double* ky; /* latency_ms */
} orc_profiles;

double orc_eval_dual(int n, int m, const double* s, const double* c, const double* alpha,
                     int32_t* counts, int32_t* model_of, orc_counters* ctr);

/* Returns 0 ok; nonzero = the reference would throw ValidationError. */
int orc_solve_dual(int n, int m, const double* s, const double* c, const orc_sub_params* p,
                   const double* init_alpha, double* alpha_star, double* score,
                   double* dual_bound, double* gap, int32_t* assignment, double* residual,
                   int32_t* iterations, int32_t* converged, orc_counters* ctr);

int orc_project_simplex(int m, const double* v, double* w);

double orc_latency_at(const orc_profiles* lib, int prof, double load);
double orc_latency_slope(const orc_profiles* lib, int prof, double load);

/* system_latency_eval + grad for one setup (prof_idx[m]). */
void orc_system_latency_eval(const orc_profiles* lib, const int32_t* prof_idx, int m,
                             const double* w, double lambda, double kappa, double* latency,
                             double* loads, double* lats, int32_t* oor);
void orc_system_latency_grad(const orc_profiles* lib, const int32_t* prof_idx, int m,
                             const double* w, double lambda, double* grad);

typedef struct {
  double objective, score, latency_ms;
  int32_t iterations, converged;
} orc_relaxed;

int orc_optimize_fractions(int n, int m, const double* s, const orc_profiles* lib,
                           const int32_t* prof_idx, double beta, const orc_ctx* ctx,
                           const orc_pga_params* p, double* w_out, int32_t* oor_out,
                           orc_relaxed* out, orc_counters* ctr);

typedef struct {
  int32_t feasible, has_beta_star, n_trace;
  double beta_star;
  orc_relaxed best;
} orc_beta_result;

int orc_optimize_beta(int n, int m, const double* s, const orc_profiles* lib,
                      const int32_t* prof_idx, const orc_ctx* ctx, const orc_beta_params* p,
                      double* w_star, double* best_w, int32_t* best_oor, orc_beta_result* out,
                      int trace_cap, double* tr_beta, double* tr_score, double* tr_lat,
                      int32_t* tr_ok, orc_counters* ctr);

/* select_setup's per-setup `evaluate` (setup_search.cpp:187-211). */
typedef struct {
  int32_t feasible;
  double score, latency_ms, beta;
} orc_setup_eval;

int orc_evaluate_setup(int n, int m, const double* s, const orc_profiles* lib,
                       const int32_t* prof_idx, const orc_ctx* ctx, const orc_beta_params* p,
                       orc_setup_eval* out, double* w_out, int32_t* oor_out, orc_counters* ctr);

/* Order-deterministic reduction (setup_search.cpp:246-253); returns best k or -1. */
int64_t orc_reduce(int64_t count, const int32_t* feasible, const double* score,
                   const double* latency);

#ifdef __cplusplus
}
#endif
#endif
