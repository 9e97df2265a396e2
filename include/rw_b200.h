/* rw_b200.h — C-ABI of the B200-native RouterWise setup-search inner loop.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++ or
 * torch types.  Every entry point replaces one function of the reference C++ solver
 * API (/root/reference/proj/include/routeplan/...); the replaced interface is cited on
 * each declaration.  INTEGRATION.md shows the C++ forwarding shim a maintainer adds so
 * the reference's host code (runner.cpp:46-58 `run_search`) links against this.
 *
 * Conventions
 *  - scores: row-major N x M doubles, `scores[j * M + i]` (workload.hpp:15).
 *  - model order is the score-matrix column order (setup_search.cpp:160-161).
 *  - latency profiles: CSR table; profile p has knots [knot_offsets[p], knot_offsets[p+1])
 *    with strictly increasing load, first load 0 after ingestion (latency.cpp:82-138, anchored at :133-134).
 *    A setup names one profile per model (`profile_index[k * M + i]`), i.e. the
 *    (model, tp, round(rho*1e4), metric) key lookup of latency.cpp:12, 60-62 is resolved by
 *    the host before the call.
 *  - all calls are synchronous w.r.t. the host unless stated; results are bit-identical to
 *    the reference CPU solver.
 *  - errors: every function returns an rw_status; the message is available from
 *    rw_last_error(ctx).  RW_ERR_VALIDATION / RW_ERR_CONFIG carry the same text the
 *    reference's ValidationError / ConfigError would (errors.hpp:9-18).
 *  - M <= RW_MAX_MODELS (device register tiles); larger M returns RW_ERR_UNSUPPORTED.
 */
#ifndef RW_B200_H
#define RW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RW_ABI_VERSION 1
#define RW_MAX_MODELS 32
#define RW_MAX_TRACE 128

typedef enum {
  RW_OK = 0,
  RW_ERR_VALIDATION = 1,  /* routeplan::ValidationError */
  RW_ERR_CONFIG = 2,      /* routeplan::ConfigError */
  RW_ERR_CUDA = 3,
  RW_ERR_NCCL = 4,
  RW_ERR_UNSUPPORTED = 5
} rw_status;

typedef struct rw_ctx rw_ctx; /* owns device buffers + a stream on one GPU */

/* score_dual.hpp:41-47 SubgradientParams (init_alpha passed separately). */
typedef struct {
  double eta0;
  int32_t max_iters;
  double residual_tol;
  int32_t polish_passes;
} rw_subgradient_params;

/* routing_opt.hpp:27-34 PgaParams (no on_iterate hook). */
typedef struct {
  double eta;
  int32_t max_iters;
  double w_tol;
  rw_subgradient_params dual;
} rw_pga_params;

/* routing_opt.hpp:60-65 BetaSearchParams. */
typedef struct {
  double beta_min;
  double beta_max; /* < 0 -> 10 / tau */
  double epsilon;  /* < 0 -> (beta_max - beta_min) / 1024 */
  rw_pga_params pga;
} rw_beta_params;

/* routing_opt.hpp:18-25 OptimizeContext minus the pointers (scores/profiles live in ctx). */
typedef struct {
  double lambda_rps;
  double tau_ms;
  double kappa;
} rw_opt_context;

/* score_dual.hpp:49-58 DualSolution (+ realised per-model counts after repair). */
typedef struct {
  double alpha_star[RW_MAX_MODELS];
  double count_residual[RW_MAX_MODELS];
  int32_t counts[RW_MAX_MODELS];
  double score;
  double dual_bound;
  double duality_gap;
  int32_t iterations;
  int32_t converged;
  int64_t eval_passes; /* eval_dual-equivalent passes executed (SURVEY §8d "evals") */
} rw_dual_solution;

/* routing_opt.hpp:36-44 RelaxedSolveResult. out_of_range is a bit mask over models. */
typedef struct {
  double w[RW_MAX_MODELS];
  double objective;
  double score;
  double latency_ms;
  int32_t iterations;
  int32_t converged;
  uint32_t out_of_range;
  int32_t pad_;
  int64_t eval_passes;
} rw_relaxed_result;

/* routing_opt.hpp:53-58 BetaStep. */
typedef struct {
  double beta;
  double score;
  double latency_ms;
  int32_t feasible;
  int32_t pad_;
} rw_beta_step;

/* routing_opt.hpp:67-73 BetaSearchResult (trace returned separately). */
typedef struct {
  int32_t feasible;
  int32_t has_beta_star;
  double beta_star;
  double w_star[RW_MAX_MODELS];
  rw_relaxed_result best;
  int32_t n_trace;
  int32_t pad_;
  int64_t eval_passes;
} rw_beta_result;

/* One retained setup's outcome: the `Eval` of setup_search.cpp:177-184 plus the sweep
 * record id (setup_search.hpp:45-51) and instrumentation.  Fixed size so records can be
 * gathered across GPUs with one collective. */
typedef struct {
  int64_t setup_id;
  int32_t feasible;
  int32_t status; /* rw_status of this setup's solve */
  double score;
  double latency_ms;
  double beta;
  double tau_ms; /* the SLO this record was solved for */
  double w[RW_MAX_MODELS];
  uint32_t out_of_range;
  int32_t bisect_steps;
  int64_t eval_passes;   /* eval_dual passes of the reference's trajectory (parity) */
  int64_t polish_passes;
  int64_t repair_calls;
  int64_t exec_passes;   /* eval passes the GPU executed (memoised solves excluded);
                            the throughput metric counts these */
} rw_setup_record;

/* ---- lifecycle ------------------------------------------------------------------- */
int rw_abi_version(void);
/* CUDA devices visible to this process (0 when none). */
int rw_device_count(void);
int rw_create(int device, rw_ctx** out);
void rw_destroy(rw_ctx* ctx);
/* Last error message of ctx (or of the calling thread when ctx is NULL). */
const char* rw_last_error(const rw_ctx* ctx);
/* Launch all work on this cudaStream_t (NULL = the ctx's own stream). */
int rw_set_stream(rw_ctx* ctx, void* cuda_stream);
/* Device time of the last solver kernel launch (CUDA events on the launch stream). */
int rw_last_kernel_ms(const rw_ctx* ctx, double* ms);

/* Diagnostics: counters summed over CTAs and over the launches since the last read
 * (RW_PROF_SLOTS entries; see rw_solver.cuh `Prof` for the slot meanings: pass phase
 * cycles, block classification counts, walker cycles, polish cycles and misses). */
#define RW_PROF_SLOTS 32
int rw_set_profiling(rw_ctx* ctx, int enable);
int rw_get_profile(rw_ctx* ctx, int64_t* out);
/* Diagnostics: `passes` eval passes at fixed prices on one CTA (per-pass cost probe). */
int rw_bench_passes(rw_ctx* ctx, const double* targets, const double* alpha, int32_t passes,
                    double* g);

/* ---- inputs ------------------------------------------------------------------------ */
/* Copy the N x M score matrix from host memory into the ctx's HBM buffer
 * (replaces ScoreMatrix ownership, workload.hpp:12-23; values validated like
 * ScoreMatrix::validate, workload.cpp:12-30).  The copy is enqueued on the ctx stream and
 * the call returns without waiting for it: from page-locked (pinned) memory it overlaps
 * whatever runs before it on the stream; the caller keeps host_scores unchanged until the
 * next synchronising call (rw_sweep_fetch, any solver entry point). */
int rw_load_scores(rw_ctx* ctx, int32_t n, int32_t m, const double* host_scores);
/* Borrow an already-resident device matrix (caller keeps it alive). */
int rw_bind_scores_device(rw_ctx* ctx, int32_t n, int32_t m, const double* device_scores);
/* Upload the latency profile table (replaces ProfileLibrary, latency.hpp:36-42;
 * validated like LatencyProfile::validate, latency.cpp:39-51). */
int rw_load_profiles(rw_ctx* ctx, int32_t n_profiles, const int64_t* knot_offsets,
                     const double* knot_load, const double* knot_latency);

/* ---- solver entry points (one setup / one price vector) ---------------------------- */
/* score_dual.hpp:38-39 dual_objective(scores, targets, prices). */
int rw_dual_objective(rw_ctx* ctx, const double* targets, const double* alpha, double* g);
/* score_dual.hpp:34 assign_prompts(scores, prices); m_alpha must equal M. */
int rw_assign_prompts(rw_ctx* ctx, int32_t m_alpha, const double* alpha, int32_t* model_of,
                      int32_t* counts);
/* score_dual.hpp:64-65 solve_dual(scores, targets, params); init_alpha may be NULL.
 * assignment (N ints) may be NULL. */
int rw_solve_dual(rw_ctx* ctx, const double* targets, const rw_subgradient_params* params,
                  const double* init_alpha, rw_dual_solution* out, int32_t* assignment);
/* The chosen setup's routing policy {alpha*, counts, assignment}.  PlanResult carries only
 * w* (setup_search.hpp:53-65); the reference re-derives the policy with a cold
 * solve_dual(scores, counts_for(w*)) (test_cli.cpp:103-106), which is optimize_fractions'
 * canonical final solve at the winning iterate (routing_opt.cpp:121-123).  Targets are
 * c_i = N * w_i exactly as counts_for (routing_opt.cpp:28-33).  m must equal M;
 * assignment (N ints) may be NULL. */
int rw_winner_policy(rw_ctx* ctx, int32_t m, const double* w_star,
                     const rw_subgradient_params* params, rw_dual_solution* out,
                     int32_t* assignment);
/* routing_opt.hpp:15 project_simplex(v). Runs the device routine on one vector. */
int rw_project_simplex(rw_ctx* ctx, int32_t m, const double* v, double* w);
/* latency.hpp:59-77 system_latency_eval + system_latency_grad for one setup. */
int rw_system_latency_eval(rw_ctx* ctx, const int32_t* profile_index, const double* w,
                           double lambda_rps, double kappa, double* latency_ms,
                           double* per_model_load, double* per_model_latency,
                           int32_t* out_of_range, double* grad);
/* routing_opt.hpp:50-51 optimize_fractions(setup, beta, ctx, params). */
int rw_optimize_fractions(rw_ctx* ctx, const int32_t* profile_index, double beta,
                          const rw_opt_context* opt, const rw_pga_params* params,
                          rw_relaxed_result* out);
/* routing_opt.hpp:79-80 optimize_beta(setup, ctx, params); trace may be NULL. */
int rw_optimize_beta(rw_ctx* ctx, const int32_t* profile_index, const rw_opt_context* opt,
                     const rw_beta_params* params, rw_beta_result* out, int32_t trace_cap,
                     rw_beta_step* trace);

/* ---- the sweep (setup_search.cpp:154-272, per-setup half) --------------------------- */
/* Solve every retained setup k with k % shard_count == shard_rank (interleaved sharding,
 * SURVEY §8e) on this GPU in one persistent kernel; writes one record per solved setup, in
 * increasing k, to out_records (capacity >= ceil(n_setups / shard_count)).
 * profile_index is n_setups x M; setup_ids are the enumeration ordinals. */
int rw_sweep(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids,
             const int32_t* profile_index, const rw_opt_context* opt,
             const rw_beta_params* params, int32_t shard_rank, int32_t shard_count,
             rw_setup_record* out_records, int64_t* n_out);
/* SLO sweep: every (setup, tau) pair of n_setups x n_slo is one independent instance
 * (the reference takes one tau per select_setup call; this batches them in one launch).
 * Instance k = slo * n_setups + setup; sharding is over k.  opt->tau_ms is ignored;
 * params[t] are SLO t's search parameters (n_slo entries). */
int rw_sweep_slo(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids,
                 const int32_t* profile_index, int32_t n_slo, const double* tau_ms,
                 const rw_opt_context* opt, const rw_beta_params* params, int32_t shard_rank,
                 int32_t shard_count, rw_setup_record* out_records, int64_t* n_out);
/* Asynchronous variants: enqueue the sweep on the ctx's stream and return without waiting
 * for the device (the next step's uploads overlap the running kernel).  setup_ids, tau_ms
 * and params are staged through a context-owned host buffer and may be reused at once;
 * profile_index, when page-locked, must stay unchanged until rw_sweep_fetch.  Records stay
 * in device memory (ctx-owned, or the rw_set_records_device buffer) until rw_sweep_fetch. */
int rw_sweep_async(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids,
                   const int32_t* profile_index, const rw_opt_context* opt,
                   const rw_beta_params* params, int32_t shard_rank, int32_t shard_count);
int rw_sweep_slo_async(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids,
                       const int32_t* profile_index, int32_t n_slo, const double* tau_ms,
                       const rw_opt_context* opt, const rw_beta_params* params,
                       int32_t shard_rank, int32_t shard_count);
int rw_sweep_fetch(rw_ctx* ctx, rw_setup_record* out_records, int64_t* n_out);
/* Let subsequent sweeps write their records into a caller-owned DEVICE buffer of
 * cap_records records on the ctx's GPU (NULL = back to the ctx-owned buffer).  The records
 * then never leave HBM before the cross-GPU exchange: one all-gather of these fixed-size
 * buffers over NCCL/NVLink, e.g. torch.distributed.all_gather_into_tensor.
 * rw_sweep_fetch still works (it reads from this buffer). */
int rw_set_records_device(rw_ctx* ctx, void* device_records, int64_t cap_records);

/* select_setup's per-setup half over several GPUs (SearchParams::parallelism,
 * setup_search.hpp:74-77, mapped to GPUs): one host thread per context, shard r of W =
 * n_ctx solved on ctxs[r] (instances k with k % W == r), each context
 * holding its own replica of the scores and profiles.  The fixed-size records come back
 * in instance order (k = slo * n_setups + setup), so the result is bit-identical to a
 * single-GPU rw_sweep_slo; out_records holds n_setups * n_slo records.  Errors: the first
 * failing shard in rank order (the reference rethrows worker failures in thread order,
 * setup_search.cpp:230-235); its message is set on ctxs[0]. */
int rw_sweep_multi(rw_ctx* const* ctxs, int32_t n_ctx, int64_t n_setups,
                   const int64_t* setup_ids, const int32_t* profile_index, int32_t n_slo,
                   const double* tau_ms, const rw_opt_context* opt,
                   const rw_beta_params* params, rw_setup_record* out_records);

/* f4: the same sweep with a speculative beta bisection.  optimize_beta
 * (routing_opt.cpp:138-173) is sequential; each round here evaluates the next `depth`
 * levels of every instance's bisection tree in one launch (depth 2: the midpoint and both
 * midpoints the next step can take) and the host follows the realised path with the
 * reference's bracket arithmetic.  Records are bit-identical to rw_sweep_slo's (same
 * eval_passes = the reference trajectory's); exec_passes also counts the discarded
 * branches.  For sweeps too small to fill the GPU (C1: 64 setups) it cuts the sequential
 * depth of the default schedule's 10-11 bisection steps to 6 rounds.  depth 1..4;
 * out_records holds n_setups * n_slo records in instance order. */
int rw_sweep_spec(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids,
                  const int32_t* profile_index, int32_t n_slo, const double* tau_ms,
                  const rw_opt_context* opt, const rw_beta_params* params, int32_t depth,
                  rw_setup_record* out_records, int64_t* n_out);

/* Order-deterministic winner (setup_search.cpp:246-253): feasible, max score, then min
 * latency, then smallest setup_id.  Records may come from any number of shards in any
 * order.  Returns the record index or -1. */
int64_t rw_reduce_records(int64_t n, const rw_setup_record* records);

/* ---- f2: binary score files ------------------------------------------ */
/* The reference reads scores from CSV (load_scores, workload.cpp:32-62).  A .f64 score
 * file ("RWSCORE1" | int64 n | int64 m | m x (int32 len, name) | n*m float64 row-major)
 * is one read; pair it with rw_load_scores from a pinned buffer for an asynchronous H2D.
 * Entries are validated like ScoreMatrix::validate (workload.cpp:23-29); a missing or
 * malformed file is RW_ERR_CONFIG (the reference's ConfigError for inputs).  Messages:
 * rw_host_last_error(). */
int rw_write_scores_f64(const char* path, int64_t n, int32_t m, const char* const* models,
                        const double* scores);
/* out == NULL: header only (n, m, names '\0'-separated into names[names_cap]). */
int rw_read_scores_f64(const char* path, int64_t* n, int32_t* m, double* out, int64_t out_cap,
                       char* names, int64_t names_cap);
const char* rw_host_last_error(void);

/* ---- host-side input producers ------------------------------------------------------ */
/* workload.cpp:78-112 synth_scores: Beta(a_i, b_i) columns via mt19937_64 + libstdc++
 * gamma_distribution, model-major draw order; identical matrix on this platform. */
int rw_synth_scores(int32_t n, int32_t m, const double* shape_a, const double* shape_b,
                    uint64_t seed, double* out);

/* setup_search.cpp:99-152 enumerate_setups + retain.  Choices per model in CSR form,
 * memory table entries (model, tp, fraction).  name_rank[i] is model i's rank in byte-wise
 * name order (FFD breaks size ties by model name, setup_search.cpp:76-79); NULL = index order.
 * Writes verdict per enumerated setup
 * (0 RETAINED, 1 UNDER_UTILIZED, 2 OVER_BUDGET, 3 PLACEMENT_INFEASIBLE) and its (tp, rho)
 * per model, up to cap setups; *n_enumerated gets the total. */
int rw_enumerate_retain(int32_t m, const int32_t* name_rank, const int32_t* tp_offsets,
                        const int32_t* tp_values, const int32_t* rho_offsets,
                        const double* rho_values, int32_t n_mem, const int32_t* mem_model,
                        const int32_t* mem_tp, const double* mem_fraction, int32_t gpu_count,
                        double rho_floor,
                        int64_t cap, int64_t* n_enumerated, int32_t* verdict, int32_t* tp_out,
                        double* rho_out);

#ifdef __cplusplus
}
#endif
#endif /* RW_B200_H */
