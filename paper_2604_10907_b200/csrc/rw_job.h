// Job descriptor shared by the host ABI (rw_abi.cpp) and the device solver (rw_solver.cuh).
// Passed by value as the kernel parameter; every pointer is device memory.
#pragma once
#include <cuda.h>  // CUtensorMap (header only; the encoder is fetched through the runtime)
#include <stdint.h>

#include "rw_b200.h"

namespace rw {

enum JobKind : int32_t {
  JOB_EVAL = 0,     // one priced pass: g, counts, assignment   (dual_objective / assign_prompts)
  JOB_SOLVE = 1,    // solve_dual
  JOB_OPTFRAC = 2,  // optimize_fractions
  JOB_OPTBETA = 3,  // optimize_beta
  JOB_SWEEP = 4,    // select_setup per-setup evaluate, persistent over a work queue
  JOB_SIMPLEX = 5,  // project_simplex on one vector
  JOB_LATENCY = 6,  // system_latency_eval + grad for one setup
  JOB_BENCH_PASS = 7,  // diagnostics: trace_cap eval passes at fixed prices
  JOB_FRAC_BATCH = 8,  // optimize_fractions over (setup, SLO, beta) items (speculative bisection)
};

// One optimize_fractions evaluation of a speculative beta bisection (rw_sweep_spec).
struct FracItem {
  int32_t setup;  // index into the sweep's setups
  int32_t slo;    // index into taus / bps
  double beta;
};
struct FracRecord {  // routing_opt.hpp:36-44 RelaxedSolveResult + counters
  double w[RW_MAX_MODELS];
  double score, latency_ms, objective;
  int32_t iterations, converged;
  uint32_t out_of_range;
  int32_t status;
  int64_t eval_passes, polish_passes, repair_calls, exec_passes;
};

struct Job {
  // 2-D tiled TMA descriptor of the score matrix (box = one ring stage of SR rows, with the
  // 32/64/128-byte smem swizzle matching the row width), for M in {4, 8, 16}; the kernel
  // takes the Job as a __grid_constant__ parameter so the descriptor lives in param space.
  alignas(64) CUtensorMap tmap;
  int32_t tmap_ok;
  int32_t kind;
  int32_t n, m;
  const double* scores;
  // latency profile table (CSR)
  const int64_t* koff;
  const double* kx;
  const double* ky;
  // setups
  const int32_t* prof_idx;  // [n_items * m]
  const int64_t* setup_ids;
  int64_t n_items;      // instances = n_setups * n_slo
  int64_t n_setups;
  const double* taus;   // [n_slo] (JOB_SWEEP); null -> opt.tau_ms
  const rw_beta_params* bps;  // [n_slo] per-SLO params (JOB_SWEEP); null -> bp
  int32_t shard_rank, shard_count;
  rw_opt_context opt;
  rw_beta_params bp;
  double beta;                  // JOB_OPTFRAC
  double c[RW_MAX_MODELS];      // targets (EVAL, SOLVE)
  double vec[RW_MAX_MODELS];    // alpha (EVAL), init_alpha (SOLVE), v (SIMPLEX), w (LATENCY)
  int32_t has_vec;
  int32_t trace_cap;
  // outputs
  rw_setup_record* records;
  rw_dual_solution* dual_out;
  rw_relaxed_result* relaxed_out;
  rw_beta_result* beta_out;
  rw_beta_step* trace_out;
  int32_t* assign_out;  // [n]
  double* dvec_out;     // EVAL: {g}; SIMPLEX: w[m]; LATENCY: {lat, loads[m], lats[m], grad[m]}
  int32_t* ivec_out;    // EVAL: counts[m]; LATENCY: oor[m]
  int32_t* status_out;  // job-level status (first error)
  char* msg_out;        // job-level message buffer (256 bytes)
  // workspace, one slot of n entries per CTA
  uint8_t* ws_model_of;
  // repair Phase-2 pair lists, one slot of ph2_stride bytes per CTA (Solver::ph2_ws)
  unsigned char* ws_ph2;
  long long ph2_stride;
  int32_t ph2_k, ph2_ec;
  unsigned long long* queue;
  long long* prof_out;  // optional diagnostics counters [RW_PROF_SLOTS]
  // JOB_FRAC_BATCH
  const FracItem* frac_items;  // [n_items]
  FracRecord* frac_out;        // [n_items]
};

// Repair Phase-2 list geometry for m models: K best members per pair (<= the 2048-pair
// sort buffer), EC joined rows per pair, about 1 MB per CTA slot.
inline int ph2_ec(int m) { (void)m; return 64; }
inline int ph2_k(int m) {
  const long long pairs = (long long)m * m;
  long long k = (1ll << 20) / (pairs * 12) - ph2_ec(m);
  return (int)(k < 16 ? 16 : (k > 2048 ? 2048 : k));
}
inline long long ph2_stride(int m) {
  const long long pairs = (long long)m * m;
  long long b = pairs * (ph2_k(m) + ph2_ec(m)) * 12 + pairs * 24;
  return (b + 255) / 256 * 256;
}

// Rows per TMA ring stage of the kernel instantiated for m models (Smem<MM,...>::SR).
inline int stage_rows(int m) { return m <= 4 ? 128 : (m <= 8 ? 64 : 32); }
// M for which the eval / polish streams use the swizzled tensor-map copies.
inline bool swizzled_m(int m) { return m == 4 || m == 8 || m == 16; }

// Host launcher (rw_kernels.cu). Returns a cudaError_t value.
int launch_job(const Job& job, int grid, void* stream);
// Largest number of CTAs the sweep kernel keeps resident for this (m) on `device`.
int sweep_max_resident(int m, int device);

}  // namespace rw
