// Job descriptor shared by the host ABI (rw_abi.cpp) and the device solver (rw_solver.cuh).
// Passed by value as the kernel parameter; every pointer is device memory.
#pragma once
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
};

struct Job {
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
  unsigned long long* queue;
  long long* prof_out;  // optional diagnostics counters [RW_PROF_SLOTS]
};

// Host launcher (rw_kernels.cu). Returns a cudaError_t value.
int launch_job(const Job& job, int grid, void* stream);
// Largest number of CTAs the sweep kernel keeps resident for this (m) on `device`.
int sweep_max_resident(int m, int device);

}  // namespace rw
