// rw_abi.cpp — the C-ABI (include/rw_b200.h): context, input upload, validation with the
// reference's error texts, job launch and result download.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rw_b200.h"
#include "rw_job.h"

struct rw_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // scores
  const double* d_scores = nullptr;
  double* d_scores_owned = nullptr;
  size_t scores_cap = 0;  // doubles
  int32_t n = 0, m = 0;
  CUtensorMap tmap;        // 2-D TMA descriptor of the scores (swizzled_m(m) only)
  bool tmap_ok = false;
  // profiles
  int64_t* d_koff = nullptr;
  double* d_kx = nullptr;
  double* d_ky = nullptr;
  int32_t n_prof = 0;
  std::vector<int64_t> h_koff;
  // workspace
  uint8_t* d_mo = nullptr;
  size_t ws_entries = 0;  // slots * n capacity
  unsigned char* d_ph2 = nullptr;  // repair Phase-2 lists, slots * ph2_stride(m)
  size_t ph2_bytes = 0;
  // generic io
  void* d_io = nullptr;
  size_t io_cap = 0;
  unsigned long long* d_queue = nullptr;
  int32_t* d_status = nullptr;
  // sweep
  int32_t* d_prof_idx = nullptr;
  size_t prof_idx_cap = 0;
  int64_t* d_setup_ids = nullptr;
  size_t setup_ids_cap = 0;
  rw_setup_record* d_records = nullptr;
  size_t records_cap = 0;
  rw_setup_record* d_records_user = nullptr;  // caller-owned device buffer (optional)
  int64_t records_user_cap = 0;
  int64_t pending_records = -1;
  std::vector<unsigned char> h_stage;  // pageable staging of per-sweep tables
  // speculative bisection (rw_sweep_spec)
  void* d_items = nullptr;
  size_t items_cap = 0;
  void* d_frac = nullptr;
  size_t frac_cap = 0;
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timed = false;
  long long* d_prof = nullptr;  // optional cycle counters (rw_set_profiling)
  std::string err;
};

namespace {

thread_local std::string g_tls_err;

int set_err(rw_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_tls_err = msg;
  return code;
}

int cuda_err(rw_ctx* ctx, cudaError_t e, const char* where) {
  return set_err(ctx, RW_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                              \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_err(ctx, e_, #call);   \
  } while (0)

// The driver's tensor-map encoder, fetched through the runtime (no libcuda link).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// (Re)build the score matrix's tensor map: dims {M, N} doubles, row pitch 8M bytes, box
// {M, SR} = one ring stage, smem swizzle = the row width (32/64/128 B), zero fill past N.
int encode_scores_map(rw_ctx* ctx) {
  ctx->tmap_ok = false;
  if (!rw::swizzled_m(ctx->m)) return RW_OK;
  auto enc = tensor_map_encoder();
  if (!enc) return set_err(ctx, RW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)ctx->m, (cuuint64_t)ctx->n};
  const cuuint64_t strides[1] = {(cuuint64_t)ctx->m * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)ctx->m, (cuuint32_t)rw::stage_rows(ctx->m)};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle swz = ctx->m == 4 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : ctx->m == 8 ? CU_TENSOR_MAP_SWIZZLE_64B
                                               : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(&ctx->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                   const_cast<double*>(ctx->d_scores), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(ctx, RW_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  ctx->tmap_ok = true;
  return RW_OK;
}

// libstdc++'s std::to_string(double) (the reference builds its messages with it).
std::string dstr(double x) { return std::to_string(x); }

int ensure(rw_ctx* ctx, void** p, size_t* cap, size_t bytes) {
  if (*cap >= bytes && *p) return RW_OK;
  CK(cudaSetDevice(ctx->device));  // allocations land on the ctx's GPU
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  size_t b = std::max<size_t>(bytes, 256);
  CK(cudaMalloc(p, b));
  *cap = b;
  return RW_OK;
}

int ensure_ws(rw_ctx* ctx, int slots) {
  size_t need = (size_t)slots * (size_t)ctx->n;
  const size_t ph2 = (size_t)slots * (size_t)rw::ph2_stride(ctx->m > 0 ? ctx->m : 1);
  if (ctx->ph2_bytes < ph2 || !ctx->d_ph2) {
    CK(cudaSetDevice(ctx->device));
    if (ctx->d_ph2) cudaFree(ctx->d_ph2);
    ctx->d_ph2 = nullptr;
    ctx->ph2_bytes = 0;
    CK(cudaMalloc(&ctx->d_ph2, ph2));
    ctx->ph2_bytes = ph2;
  }
  if (ctx->ws_entries >= need && ctx->d_mo) return RW_OK;
  CK(cudaSetDevice(ctx->device));
  if (ctx->d_mo) cudaFree(ctx->d_mo);
  ctx->d_mo = nullptr;
  ctx->ws_entries = 0;
  CK(cudaMalloc(&ctx->d_mo, std::max<size_t>(need, 1) + 64));  // +64: 16-byte tail loads
  ctx->ws_entries = need;
  return RW_OK;
}

int need_inputs(rw_ctx* ctx, bool profiles) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (!ctx->d_scores || ctx->n <= 0 || ctx->m <= 0)
    return set_err(ctx, RW_ERR_VALIDATION, "score matrix is empty");
  if (ctx->m > RW_MAX_MODELS)
    return set_err(ctx, RW_ERR_UNSUPPORTED,
                   "rw_b200 supports at most " + std::to_string(RW_MAX_MODELS) + " models");
  if (profiles && !ctx->d_koff)
    return set_err(ctx, RW_ERR_VALIDATION, "optimizer context: missing scores or profiles");
  CK(cudaSetDevice(ctx->device));
  return RW_OK;
}

// TargetCounts::validate (score_dual.cpp:195-205)
int validate_targets(rw_ctx* ctx, const double* c) {
  for (int i = 0; i < ctx->m; ++i)
    if (!std::isfinite(c[i]) || c[i] < -1e-9)
      return set_err(ctx, RW_ERR_VALIDATION,
                     "target counts: entry " + std::to_string(i) + " is negative");
  double t = 0.0;
  for (int i = 0; i < ctx->m; ++i) t += c[i];
  if (std::abs(t - ctx->n) > 1e-6 * std::max(1.0, static_cast<double>(ctx->n)))
    return set_err(ctx, RW_ERR_VALIDATION,
                   "target counts sum to " + dstr(t) + ", expected " + std::to_string(ctx->n));
  return RW_OK;
}

int validate_profile_index(rw_ctx* ctx, const int32_t* pidx, size_t count) {
  for (size_t k = 0; k < count; ++k)
    if (pidx[k] < 0 || pidx[k] >= ctx->n_prof)
      return set_err(ctx, RW_ERR_CONFIG,
                     "no latency profile for index " + std::to_string(pidx[k]));
  return RW_OK;
}

rw::Job base_job(rw_ctx* ctx, int kind) {
  rw::Job j;
  std::memset(&j, 0, sizeof(j));
  j.kind = kind;
  j.tmap = ctx->tmap;
  j.tmap_ok = ctx->tmap_ok ? 1 : 0;
  j.n = ctx->n;
  j.m = ctx->m;
  j.scores = ctx->d_scores;
  j.koff = ctx->d_koff;
  j.kx = ctx->d_kx;
  j.ky = ctx->d_ky;
  j.shard_count = 1;
  j.ws_model_of = ctx->d_mo;
  j.ws_ph2 = ctx->d_ph2;
  j.ph2_stride = rw::ph2_stride(ctx->m > 0 ? ctx->m : 1);
  j.ph2_k = rw::ph2_k(ctx->m > 0 ? ctx->m : 1);
  j.ph2_ec = rw::ph2_ec(ctx->m);
  j.queue = ctx->d_queue;
  j.status_out = ctx->d_status;
  j.prof_out = ctx->d_prof;
  return j;
}

// Launch + time + wait; maps device status to an error.
int run(rw_ctx* ctx, rw::Job& j, int grid) {
  // every launch goes to the ctx's GPU, whatever device the calling thread had current
  CK(cudaSetDevice(ctx->device));
  if (rw::swizzled_m(j.m) && j.n > 0 && !j.tmap_ok)  // the kernel has no other load path
    return set_err(ctx, RW_ERR_CUDA, "score tensor map missing");
  j.ws_model_of = ctx->d_mo;
  j.ws_ph2 = ctx->d_ph2;
  CK(cudaMemsetAsync(ctx->d_status, 0, sizeof(int32_t), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_queue, 0, sizeof(unsigned long long), ctx->stream));
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  int e = rw::launch_job(j, grid, ctx->stream);
  if (e != 0) return cuda_err(ctx, (cudaError_t)e, "solver_kernel launch");
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->timed = true;
  return RW_OK;
}

int finish(rw_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  int32_t st = 0;
  CK(cudaMemcpy(&st, ctx->d_status, sizeof(st), cudaMemcpyDeviceToHost));
  if (st == RW_ERR_VALIDATION)
    return set_err(ctx, RW_ERR_VALIDATION,
                   "solver: invalid intermediate state (non-finite or inconsistent targets)");
  if (st) return set_err(ctx, st, "solver: device status " + std::to_string(st));
  return RW_OK;
}

}  // namespace

extern "C" {

int rw_abi_version(void) { return RW_ABI_VERSION; }

int rw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int rw_create(int device, rw_ctx** out) {
  if (!out) return set_err(nullptr, RW_ERR_VALIDATION, "rw_create: null out");
  *out = nullptr;
  rw_ctx* ctx = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_err(nullptr, e, "cudaSetDevice");
  ctx = new rw_ctx();
  ctx->device = device;
#define CKC(call)                          \
  do {                                     \
    cudaError_t e2 = (call);               \
    if (e2 != cudaSuccess) {               \
      int rc = cuda_err(nullptr, e2, #call); \
      rw_destroy(ctx);                     \
      return rc;                           \
    }                                      \
  } while (0)
  CKC(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  CKC(cudaEventCreate(&ctx->ev0));
  CKC(cudaEventCreate(&ctx->ev1));
  CKC(cudaMalloc(&ctx->d_queue, sizeof(unsigned long long)));
  CKC(cudaMalloc(&ctx->d_status, sizeof(int32_t)));
#undef CKC
  *out = ctx;
  return RW_OK;
}

void rw_destroy(rw_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->d_scores_owned);
  cudaFree(ctx->d_koff);
  cudaFree(ctx->d_kx);
  cudaFree(ctx->d_ky);
  cudaFree(ctx->d_mo);
  cudaFree(ctx->d_ph2);
  cudaFree(ctx->d_io);
  cudaFree(ctx->d_queue);
  cudaFree(ctx->d_status);
  cudaFree(ctx->d_prof_idx);
  cudaFree(ctx->d_setup_ids);
  cudaFree(ctx->d_records);
  cudaFree(ctx->d_items);
  cudaFree(ctx->d_frac);
  cudaFree(ctx->d_prof);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* rw_last_error(const rw_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_tls_err.c_str();
}

int rw_set_stream(rw_ctx* ctx, void* stream) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return RW_OK;
}

int rw_last_kernel_ms(const rw_ctx* ctx, double* ms) {
  if (!ctx || !ms || !ctx->timed) return RW_ERR_VALIDATION;
  float f = 0.f;
  if (cudaEventElapsedTime(&f, ctx->ev0, ctx->ev1) != cudaSuccess) return RW_ERR_CUDA;
  *ms = f;
  return RW_OK;
}

int rw_set_profiling(rw_ctx* ctx, int enable) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  CK(cudaSetDevice(ctx->device));
  if (enable && !ctx->d_prof) CK(cudaMalloc(&ctx->d_prof, RW_PROF_SLOTS * sizeof(long long)));
  if (!enable && ctx->d_prof) {
    cudaFree(ctx->d_prof);
    ctx->d_prof = nullptr;
  }
  if (ctx->d_prof) CK(cudaMemset(ctx->d_prof, 0, RW_PROF_SLOTS * sizeof(long long)));
  return RW_OK;
}

int rw_get_profile(rw_ctx* ctx, int64_t* out) {
  if (!ctx || !ctx->d_prof) return set_err(ctx, RW_ERR_VALIDATION, "profiling not enabled");
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(out, ctx->d_prof, RW_PROF_SLOTS * sizeof(long long), cudaMemcpyDeviceToHost));
  CK(cudaMemset(ctx->d_prof, 0, RW_PROF_SLOTS * sizeof(long long)));
  return RW_OK;
}

int rw_load_scores(rw_ctx* ctx, int32_t n, int32_t m, const double* host) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (n <= 0) return set_err(ctx, RW_ERR_VALIDATION, "score matrix: no prompts");
  if (m <= 0) return set_err(ctx, RW_ERR_VALIDATION, "score matrix: no models");
  if (m > RW_MAX_MODELS)
    return set_err(ctx, RW_ERR_UNSUPPORTED,
                   "rw_b200 supports at most " + std::to_string(RW_MAX_MODELS) + " models");
  const size_t cnt = (size_t)n * (size_t)m;
  for (size_t k = 0; k < cnt; ++k) {  // ScoreMatrix::validate (workload.cpp:23-29)
    double v = host[k];
    if (!std::isfinite(v) || v < 0.0 || v > 1.0) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", v);
      return set_err(ctx, RW_ERR_VALIDATION,
                     "score matrix: entry for prompt 'p" + std::to_string(k / m + 1) +
                         "', model " + std::to_string(k % m) + " is " + buf +
                         ", outside [0, 1]");
    }
  }
  CK(cudaSetDevice(ctx->device));
  if (ctx->scores_cap < cnt || !ctx->d_scores_owned) {
    cudaFree(ctx->d_scores_owned);
    ctx->d_scores_owned = nullptr;
    ctx->scores_cap = 0;
    CK(cudaMalloc(&ctx->d_scores_owned, cnt * sizeof(double)));
    ctx->scores_cap = cnt;
  }
  CK(cudaMemcpyAsync(ctx->d_scores_owned, host, cnt * sizeof(double), cudaMemcpyHostToDevice,
                     ctx->stream));
  ctx->d_scores = ctx->d_scores_owned;
  ctx->n = n;
  ctx->m = m;
  return encode_scores_map(ctx);
}

int rw_bind_scores_device(rw_ctx* ctx, int32_t n, int32_t m, const double* dev) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (n <= 0 || m <= 0 || !dev) return set_err(ctx, RW_ERR_VALIDATION, "score matrix is empty");
  if (m > RW_MAX_MODELS)
    return set_err(ctx, RW_ERR_UNSUPPORTED,
                   "rw_b200 supports at most " + std::to_string(RW_MAX_MODELS) + " models");
  if ((reinterpret_cast<uintptr_t>(dev) & 31u) != 0)  // 256-bit row loads
    return set_err(ctx, RW_ERR_VALIDATION, "device score matrix must be 32-byte aligned");
  ctx->d_scores = dev;
  ctx->n = n;
  ctx->m = m;
  return encode_scores_map(ctx);
}

int rw_load_profiles(rw_ctx* ctx, int32_t np, const int64_t* koff, const double* kx,
                     const double* ky) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (np <= 0) return set_err(ctx, RW_ERR_VALIDATION, "profile table: no profiles");
  if (koff[0] != 0) return set_err(ctx, RW_ERR_VALIDATION, "profile table: offsets must start at 0");
  for (int p = 0; p < np; ++p) {  // LatencyProfile::validate (latency.cpp:39-51)
    int64_t a = koff[p], b = koff[p + 1];
    std::string who = "profile " + std::to_string(p);
    if (b - a < 2) return set_err(ctx, RW_ERR_VALIDATION, who + ": needs at least two knots");
    for (int64_t k = a; k < b; ++k) {
      if (kx[k] < 0.0 || ky[k] < 0.0)
        return set_err(ctx, RW_ERR_VALIDATION, who + ": negative load or latency");
      if (k > a && !(kx[k] > kx[k - 1]))
        return set_err(ctx, RW_ERR_VALIDATION, who + ": loads must be strictly increasing");
    }
  }
  CK(cudaSetDevice(ctx->device));
  const int64_t nk = koff[np];
  cudaFree(ctx->d_koff);
  cudaFree(ctx->d_kx);
  cudaFree(ctx->d_ky);
  ctx->d_koff = nullptr;
  ctx->d_kx = ctx->d_ky = nullptr;
  CK(cudaMalloc(&ctx->d_koff, sizeof(int64_t) * (np + 1)));
  CK(cudaMalloc(&ctx->d_kx, sizeof(double) * nk));
  CK(cudaMalloc(&ctx->d_ky, sizeof(double) * nk));
  CK(cudaMemcpy(ctx->d_koff, koff, sizeof(int64_t) * (np + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_kx, kx, sizeof(double) * nk, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_ky, ky, sizeof(double) * nk, cudaMemcpyHostToDevice));
  ctx->n_prof = np;
  ctx->h_koff.assign(koff, koff + np + 1);
  return RW_OK;
}

// ---- single pass -----------------------------------------------------------------------
static int eval_job(rw_ctx* ctx, const double* targets, const double* alpha, double* g,
                    int32_t* model_of, int32_t* counts) {
  int rc;
  if ((rc = ensure_ws(ctx, 1))) return rc;
  const size_t n = ctx->n, m = ctx->m;
  size_t bytes = sizeof(double) * 4 + sizeof(int32_t) * (m + n) + 64;
  if ((rc = ensure(ctx, &ctx->d_io, &ctx->io_cap, bytes))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_EVAL);
  for (size_t i = 0; i < m; ++i) {
    j.c[i] = targets[i];
    j.vec[i] = alpha[i];
  }
  char* io = static_cast<char*>(ctx->d_io);
  j.dvec_out = reinterpret_cast<double*>(io);
  j.ivec_out = reinterpret_cast<int32_t*>(io + 32);
  j.assign_out = reinterpret_cast<int32_t*>(io + 32 + sizeof(int32_t) * m);
  if ((rc = run(ctx, j, 1))) return rc;
  if ((rc = finish(ctx))) return rc;
  if (g) CK(cudaMemcpy(g, j.dvec_out, sizeof(double), cudaMemcpyDeviceToHost));
  if (counts) CK(cudaMemcpy(counts, j.ivec_out, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
  if (model_of)
    CK(cudaMemcpy(model_of, j.assign_out, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  return RW_OK;
}

int rw_dual_objective(rw_ctx* ctx, const double* targets, const double* alpha, double* g) {
  int rc;
  if ((rc = need_inputs(ctx, false))) return rc;
  if ((rc = validate_targets(ctx, targets))) return rc;
  return eval_job(ctx, targets, alpha, g, nullptr, nullptr);
}

int rw_bench_passes(rw_ctx* ctx, const double* targets, const double* alpha, int32_t passes,
                    double* g) {
  int rc;
  if ((rc = need_inputs(ctx, false))) return rc;
  if ((rc = ensure_ws(ctx, 1))) return rc;
  if ((rc = ensure(ctx, &ctx->d_io, &ctx->io_cap, 256 + sizeof(int32_t) * ctx->m))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_BENCH_PASS);
  for (int i = 0; i < ctx->m; ++i) {
    j.c[i] = targets[i];
    j.vec[i] = alpha[i];
  }
  j.trace_cap = passes;
  char* io = static_cast<char*>(ctx->d_io);
  j.dvec_out = reinterpret_cast<double*>(io);
  j.ivec_out = reinterpret_cast<int32_t*>(io + 64);
  if ((rc = run(ctx, j, 1))) return rc;
  if ((rc = finish(ctx))) return rc;
  CK(cudaMemcpy(g, j.dvec_out, sizeof(double), cudaMemcpyDeviceToHost));
  return RW_OK;
}

int rw_assign_prompts(rw_ctx* ctx, int32_t m_alpha, const double* alpha, int32_t* model_of,
                      int32_t* counts) {
  int rc;
  if ((rc = need_inputs(ctx, false))) return rc;
  if (m_alpha != ctx->m)  // score_dual.cpp:214-216
    return set_err(ctx, RW_ERR_VALIDATION,
                   "prices have " + std::to_string(m_alpha) + " entries for " +
                       std::to_string(ctx->m) + " models");
  std::vector<double> zeros(ctx->m, 0.0);
  return eval_job(ctx, zeros.data(), alpha, nullptr, model_of, counts);
}

int rw_solve_dual(rw_ctx* ctx, const double* targets, const rw_subgradient_params* params,
                  const double* init_alpha, rw_dual_solution* out, int32_t* assignment) {
  int rc;
  if ((rc = need_inputs(ctx, false))) return rc;
  if ((rc = validate_targets(ctx, targets))) return rc;
  if (!params || !out) return set_err(ctx, RW_ERR_VALIDATION, "rw_solve_dual: null argument");
  if ((rc = ensure_ws(ctx, 1))) return rc;
  const size_t n = ctx->n, m = ctx->m;
  size_t bytes = sizeof(rw_dual_solution) + 64 + sizeof(int32_t) * n;
  if ((rc = ensure(ctx, &ctx->d_io, &ctx->io_cap, bytes))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_SOLVE);
  for (size_t i = 0; i < m; ++i) {
    j.c[i] = targets[i];
    j.vec[i] = init_alpha ? init_alpha[i] : 0.0;
  }
  j.has_vec = init_alpha ? 1 : 0;
  j.bp.pga.dual = *params;
  char* io = static_cast<char*>(ctx->d_io);
  j.dual_out = reinterpret_cast<rw_dual_solution*>(io);
  j.assign_out = reinterpret_cast<int32_t*>(io + ((sizeof(rw_dual_solution) + 63) / 64) * 64);
  if ((rc = run(ctx, j, 1))) return rc;
  if ((rc = finish(ctx))) return rc;
  CK(cudaMemcpy(out, j.dual_out, sizeof(rw_dual_solution), cudaMemcpyDeviceToHost));
  if (assignment)
    CK(cudaMemcpy(assignment, j.assign_out, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  return RW_OK;
}

int rw_winner_policy(rw_ctx* ctx, int32_t m, const double* w_star,
                     const rw_subgradient_params* params, rw_dual_solution* out,
                     int32_t* assignment) {
  int rc;
  if ((rc = need_inputs(ctx, false))) return rc;
  if (!w_star || !params || !out)
    return set_err(ctx, RW_ERR_VALIDATION, "rw_winner_policy: null argument");
  if (m != ctx->m)
    return set_err(ctx, RW_ERR_VALIDATION,
                   "routing fractions have " + std::to_string(m) + " entries for " +
                       std::to_string(ctx->m) + " models");
  std::vector<double> c(m);
  for (int i = 0; i < m; ++i) c[i] = static_cast<double>(ctx->n) * w_star[i];  // counts_for
  return rw_solve_dual(ctx, c.data(), params, nullptr, out, assignment);
}

int rw_project_simplex(rw_ctx* ctx, int32_t m, const double* v, double* w) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (m <= 0) return set_err(ctx, RW_ERR_VALIDATION, "project_simplex: empty input");
  if (m > RW_MAX_MODELS) return set_err(ctx, RW_ERR_UNSUPPORTED, "project_simplex: too many entries");
  for (int i = 0; i < m; ++i)
    if (!std::isfinite(v[i]))
      return set_err(ctx, RW_ERR_VALIDATION, "project_simplex: non-finite input");
  int rc;
  if ((rc = ensure(ctx, &ctx->d_io, &ctx->io_cap, sizeof(double) * RW_MAX_MODELS))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_SIMPLEX);
  j.n = 1;
  j.m = m;
  for (int i = 0; i < m; ++i) j.vec[i] = v[i];
  j.dvec_out = static_cast<double*>(ctx->d_io);
  if ((rc = ensure_ws(ctx, 1))) return rc;
  if ((rc = run(ctx, j, 1))) return rc;
  if ((rc = finish(ctx))) return rc;
  CK(cudaMemcpy(w, j.dvec_out, sizeof(double) * m, cudaMemcpyDeviceToHost));
  return RW_OK;
}

static int upload_pidx(rw_ctx* ctx, const int32_t* pidx, size_t count) {
  int rc;
  void* p = ctx->d_prof_idx;
  size_t cap = ctx->prof_idx_cap;
  if ((rc = ensure(ctx, &p, &cap, sizeof(int32_t) * count))) return rc;
  ctx->d_prof_idx = static_cast<int32_t*>(p);
  ctx->prof_idx_cap = cap;
  CK(cudaMemcpyAsync(ctx->d_prof_idx, pidx, sizeof(int32_t) * count, cudaMemcpyHostToDevice,
                     ctx->stream));
  return RW_OK;
}

// check_setup_and_w (latency.cpp:28-35) with RoutingFractions::validate(1e-4) (types.cpp:88-99)
static int validate_w(rw_ctx* ctx, int m, const double* w) {
  double tol = 1e-4, sum = 0.0;
  for (int i = 0; i < m; ++i) {
    if (!std::isfinite(w[i])) return set_err(ctx, RW_ERR_VALIDATION, "routing fractions: non-finite entry");
    if (w[i] < -tol) return set_err(ctx, RW_ERR_VALIDATION, "routing fractions: negative entry");
    sum += w[i];
  }
  if (std::abs(sum - 1.0) > tol)
    return set_err(ctx, RW_ERR_VALIDATION,
                   "routing fractions: entries sum to " + dstr(sum) + ", expected 1");
  for (int i = 0; i < m; ++i)
    if (w[i] < 0.0) return set_err(ctx, RW_ERR_VALIDATION, "latency_at: negative load");
  return RW_OK;
}

int rw_system_latency_eval(rw_ctx* ctx, const int32_t* pidx, const double* w, double lambda,
                           double kappa, double* latency, double* loads, double* lats,
                           int32_t* oor, double* grad) {
  int rc;
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (!ctx->d_koff) return set_err(ctx, RW_ERR_VALIDATION, "optimizer context: missing scores or profiles");
  const int m = ctx->m > 0 ? ctx->m : 0;
  if (m <= 0) return set_err(ctx, RW_ERR_VALIDATION, "score matrix is empty");
  if ((rc = validate_profile_index(ctx, pidx, m))) return rc;
  if ((rc = validate_w(ctx, m, w))) return rc;
  if ((rc = ensure(ctx, &ctx->d_io, &ctx->io_cap, sizeof(double) * (1 + 3 * m) + 4 * m + 64)))
    return rc;
  if ((rc = upload_pidx(ctx, pidx, m))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_LATENCY);
  j.prof_idx = ctx->d_prof_idx;
  for (int i = 0; i < m; ++i) j.vec[i] = w[i];
  j.opt.lambda_rps = lambda;
  j.opt.kappa = kappa;
  char* io = static_cast<char*>(ctx->d_io);
  j.dvec_out = reinterpret_cast<double*>(io);
  j.ivec_out = reinterpret_cast<int32_t*>(io + sizeof(double) * (1 + 3 * m));
  if ((rc = ensure_ws(ctx, 1))) return rc;
  if ((rc = run(ctx, j, 1))) return rc;
  if ((rc = finish(ctx))) return rc;
  std::vector<double> d(1 + 3 * m);
  std::vector<int32_t> o(m);
  CK(cudaMemcpy(d.data(), j.dvec_out, sizeof(double) * d.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(o.data(), j.ivec_out, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
  if (latency) *latency = d[0];
  for (int i = 0; i < m; ++i) {
    if (loads) loads[i] = d[1 + i];
    if (lats) lats[i] = d[1 + m + i];
    if (grad) grad[i] = d[1 + 2 * m + i];
    if (oor) oor[i] = o[i];
  }
  return RW_OK;
}

// check_context (routing_opt.cpp:11-26)
static int check_context(rw_ctx* ctx, const int32_t* pidx, const rw_opt_context* opt) {
  int rc;
  if ((rc = need_inputs(ctx, true))) return rc;
  if (!opt) return set_err(ctx, RW_ERR_VALIDATION, "optimizer context: missing");
  if (!(opt->lambda_rps > 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "arrival rate must be positive");
  if (!(opt->kappa > 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "kappa must be positive");
  return validate_profile_index(ctx, pidx, ctx->m);
}

int rw_optimize_fractions(rw_ctx* ctx, const int32_t* pidx, double beta,
                          const rw_opt_context* opt, const rw_pga_params* params,
                          rw_relaxed_result* out) {
  int rc;
  if ((rc = check_context(ctx, pidx, opt))) return rc;
  if (!(beta >= 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "beta must be >= 0");
  if (!params || !out) return set_err(ctx, RW_ERR_VALIDATION, "rw_optimize_fractions: null argument");
  if ((rc = ensure_ws(ctx, 1))) return rc;
  if ((rc = ensure(ctx, &ctx->d_io, &ctx->io_cap, sizeof(rw_relaxed_result)))) return rc;
  if ((rc = upload_pidx(ctx, pidx, ctx->m))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_OPTFRAC);
  j.prof_idx = ctx->d_prof_idx;
  j.opt = *opt;
  j.beta = beta;
  j.bp.pga = *params;
  j.relaxed_out = static_cast<rw_relaxed_result*>(ctx->d_io);
  if ((rc = run(ctx, j, 1))) return rc;
  if ((rc = finish(ctx))) return rc;
  CK(cudaMemcpy(out, j.relaxed_out, sizeof(rw_relaxed_result), cudaMemcpyDeviceToHost));
  return RW_OK;
}

static int check_beta_params(rw_ctx* ctx, const rw_opt_context* opt, const rw_beta_params* p) {
  double lo = p->beta_min, hi = p->beta_max;
  if (hi < 0.0) {  // routing_opt.cpp:143-151
    if (!(opt->tau_ms > 0.0))
      return set_err(ctx, RW_ERR_VALIDATION,
                     "latency target must be positive to derive default beta bounds");
    hi = 10.0 / opt->tau_ms;
  }
  double eps = p->epsilon;
  if (eps < 0.0) eps = (hi - lo) / 1024.0;
  if (!(lo >= 0.0) || !(lo < hi))
    return set_err(ctx, RW_ERR_VALIDATION, "beta bounds must satisfy 0 <= min < max");
  if (!(eps > 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "beta search epsilon must be positive");
  return RW_OK;
}

int rw_optimize_beta(rw_ctx* ctx, const int32_t* pidx, const rw_opt_context* opt,
                     const rw_beta_params* params, rw_beta_result* out, int32_t trace_cap,
                     rw_beta_step* trace) {
  int rc;
  if ((rc = check_context(ctx, pidx, opt))) return rc;
  if (!params || !out) return set_err(ctx, RW_ERR_VALIDATION, "rw_optimize_beta: null argument");
  if ((rc = check_beta_params(ctx, opt, params))) return rc;
  if (!trace) trace_cap = 0;
  trace_cap = std::max(0, trace_cap);
  if ((rc = ensure_ws(ctx, 1))) return rc;
  size_t bytes = sizeof(rw_beta_result) + 64 + sizeof(rw_beta_step) * (size_t)trace_cap;
  if ((rc = ensure(ctx, &ctx->d_io, &ctx->io_cap, bytes))) return rc;
  if ((rc = upload_pidx(ctx, pidx, ctx->m))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_OPTBETA);
  j.prof_idx = ctx->d_prof_idx;
  j.opt = *opt;
  j.bp = *params;
  char* io = static_cast<char*>(ctx->d_io);
  j.beta_out = reinterpret_cast<rw_beta_result*>(io);
  j.trace_out = trace_cap ? reinterpret_cast<rw_beta_step*>(
                                io + ((sizeof(rw_beta_result) + 63) / 64) * 64)
                          : nullptr;
  j.trace_cap = trace_cap;
  if ((rc = run(ctx, j, 1))) return rc;
  if ((rc = finish(ctx))) return rc;
  CK(cudaMemcpy(out, j.beta_out, sizeof(rw_beta_result), cudaMemcpyDeviceToHost));
  if (trace_cap) {
    int32_t k = std::min(trace_cap, out->n_trace);
    if (k > 0)
      CK(cudaMemcpy(trace, j.trace_out, sizeof(rw_beta_step) * k, cudaMemcpyDeviceToHost));
  }
  return RW_OK;
}

int rw_sweep_slo_async(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids,
                       const int32_t* pidx, int32_t n_slo, const double* taus,
                       const rw_opt_context* opt, const rw_beta_params* params,
                       int32_t shard_rank, int32_t shard_count) {
  int rc;
  if ((rc = need_inputs(ctx, true))) return rc;
  if (!opt || !params || !taus) return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep: null argument");
  if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
    return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep: bad shard");
  if (n_setups < 0 || n_slo < 1)
    return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep: bad setup / SLO count");
  if (!(opt->lambda_rps > 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "arrival rate must be positive");
  if (!(opt->kappa > 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "kappa must be positive");
  if (n_setups > 0) {
    for (int32_t t = 0; t < n_slo; ++t) {
      rw_opt_context o = *opt;
      o.tau_ms = taus[t];
      if ((rc = check_beta_params(ctx, &o, params + t))) return rc;
    }
    if ((rc = validate_profile_index(ctx, pidx, (size_t)n_setups * ctx->m))) return rc;
  }
  const int64_t inst = n_setups * (int64_t)n_slo;
  const int64_t items = inst > shard_rank ? (inst - shard_rank + shard_count - 1) / shard_count : 0;
  ctx->pending_records = -1;  // set only once the launch below succeeded
  if (items == 0) {
    ctx->pending_records = 0;
    return RW_OK;
  }
  CK(cudaSetDevice(ctx->device));
  if ((rc = upload_pidx(ctx, pidx, (size_t)n_setups * ctx->m))) return rc;
  {
    void* p = ctx->d_setup_ids;
    size_t cap = ctx->setup_ids_cap;
    if ((rc = ensure(ctx, &p, &cap,
                     sizeof(int64_t) * n_setups + (sizeof(double) + sizeof(rw_beta_params)) * n_slo +
                         64)))
      return rc;
    ctx->d_setup_ids = static_cast<int64_t*>(p);
    ctx->setup_ids_cap = cap;
    // one pageable staging copy of the small per-sweep tables: a pageable-source
    // cudaMemcpyAsync returns once the bytes are staged, so the call does not block on the
    // stream (the next step's uploads overlap the running kernel) and the caller's arrays —
    // even page-locked ones — may change as soon as this returns
    std::vector<unsigned char>& st = ctx->h_stage;
    const size_t b_ids = sizeof(int64_t) * n_setups, b_taus = sizeof(double) * n_slo,
                 b_par = sizeof(rw_beta_params) * n_slo;
    st.resize(b_ids + b_taus + b_par);
    if (setup_ids) {
      std::memcpy(st.data(), setup_ids, b_ids);
    } else {
      int64_t* ids = reinterpret_cast<int64_t*>(st.data());
      for (int64_t k = 0; k < n_setups; ++k) ids[k] = k;
    }
    std::memcpy(st.data() + b_ids, taus, b_taus);
    std::memcpy(st.data() + b_ids + b_taus, params, b_par);
    CK(cudaMemcpyAsync(ctx->d_setup_ids, st.data(), b_ids + b_taus + b_par,
                       cudaMemcpyHostToDevice, ctx->stream));
  }
  if (ctx->d_records_user) {
    if (ctx->records_user_cap < items)
      return set_err(ctx, RW_ERR_VALIDATION,
                     "rw_sweep: device record buffer holds " +
                         std::to_string(ctx->records_user_cap) + " records, need " +
                         std::to_string(items));
  } else {
    void* p = ctx->d_records;
    size_t cap = ctx->records_cap;
    if ((rc = ensure(ctx, &p, &cap, sizeof(rw_setup_record) * items))) return rc;
    ctx->d_records = static_cast<rw_setup_record*>(p);
    ctx->records_cap = cap;
  }
  int grid = (int)std::min<int64_t>(items, rw::sweep_max_resident(ctx->m, ctx->device));
  if ((rc = ensure_ws(ctx, grid))) return rc;
  rw::Job j = base_job(ctx, rw::JOB_SWEEP);
  j.prof_idx = ctx->d_prof_idx;
  j.setup_ids = ctx->d_setup_ids;
  j.n_items = inst;
  j.n_setups = n_setups;
  j.taus = reinterpret_cast<const double*>(ctx->d_setup_ids + n_setups);
  j.bps = reinterpret_cast<const rw_beta_params*>(ctx->d_setup_ids + n_setups + n_slo);
  j.shard_rank = shard_rank;
  j.shard_count = shard_count;
  j.opt = *opt;
  j.bp = *params;
  j.records = ctx->d_records_user ? ctx->d_records_user : ctx->d_records;
  if ((rc = run(ctx, j, grid))) return rc;
  ctx->pending_records = items;
  return RW_OK;
}

int rw_sweep_async(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids,
                   const int32_t* pidx, const rw_opt_context* opt, const rw_beta_params* params,
                   int32_t shard_rank, int32_t shard_count) {
  if (!opt) return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep: null argument");
  if (n_setups > 0 && params) {
    int rc = check_beta_params(ctx, opt, params);
    if (rc) return rc;
  }
  return rw_sweep_slo_async(ctx, n_setups, setup_ids, pidx, 1, &opt->tau_ms, opt, params,
                            shard_rank, shard_count);
}

int rw_set_records_device(rw_ctx* ctx, void* dev, int64_t cap) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (dev && cap < 1) return set_err(ctx, RW_ERR_VALIDATION, "rw_set_records_device: bad capacity");
  if (dev && (reinterpret_cast<uintptr_t>(dev) & 7u))
    return set_err(ctx, RW_ERR_VALIDATION, "rw_set_records_device: buffer must be 8-byte aligned");
  ctx->d_records_user = static_cast<rw_setup_record*>(dev);
  ctx->records_user_cap = dev ? cap : 0;
  return RW_OK;
}

int rw_sweep_fetch(rw_ctx* ctx, rw_setup_record* out, int64_t* n_out) {
  if (!ctx) return set_err(nullptr, RW_ERR_VALIDATION, "null context");
  if (ctx->pending_records < 0) return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep_fetch: no sweep");
  int64_t items = ctx->pending_records;
  ctx->pending_records = -1;
  if (n_out) *n_out = items;
  if (items == 0) return RW_OK;
  int rc = finish(ctx);
  if (rc) {
    // per-record status names the first failing setup
    std::vector<rw_setup_record> recs(items);
    cudaMemcpy(recs.data(), ctx->d_records_user ? ctx->d_records_user : ctx->d_records,
               sizeof(rw_setup_record) * items, cudaMemcpyDeviceToHost);
    for (const auto& r : recs)
      if (r.status)
        return set_err(ctx, r.status, "setup " + std::to_string(r.setup_id) + ": " + ctx->err);
    return rc;
  }
  if (out)
    CK(cudaMemcpy(out, ctx->d_records_user ? ctx->d_records_user : ctx->d_records,
                  sizeof(rw_setup_record) * items, cudaMemcpyDeviceToHost));
  return RW_OK;
}

int rw_sweep_slo(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids, const int32_t* pidx,
                 int32_t n_slo, const double* taus, const rw_opt_context* opt,
                 const rw_beta_params* params, int32_t shard_rank, int32_t shard_count,
                 rw_setup_record* out, int64_t* n_out) {
  int rc = rw_sweep_slo_async(ctx, n_setups, setup_ids, pidx, n_slo, taus, opt, params,
                              shard_rank, shard_count);
  if (rc) return rc;
  return rw_sweep_fetch(ctx, out, n_out);
}

// ---- f4: speculative beta bisection --------------------------------------------------
// optimize_beta (routing_opt.cpp:138-173) is a strictly sequential bisection: each step's
// midpoint depends on the previous step's feasibility.  A round here evaluates, for every
// instance, the next `depth` levels of the bisection tree at once (the midpoint and, for
// depth 2, both midpoints the next step can take) in ONE launch of optimize_fractions items;
// the host then walks each instance down the realised path, replaying the reference's
// bracket arithmetic and trace bookkeeping exactly (setup_search.cpp:187-211).  Same
// records, half the sequential depth at depth 2 — for sweeps too small to fill the GPU.
namespace {
struct SpecInst {
  double lo, hi, eps, tau;
  bool feasible = false, active = true;
  int n_trace = 0, status = 0;
  double tr_best_lat = 0.0, tr_best_score = 0.0, beta_star = 0.0;
  rw::FracRecord best{};
  bool degenerate = false;  // no bisection step: one optimize_fractions at beta_hi
  rw::FracRecord degen{};
  int64_t ev = 0, pol = 0, rep = 0, exec = 0;
};
}  // namespace

int rw_sweep_spec(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids, const int32_t* pidx,
                  int32_t n_slo, const double* taus, const rw_opt_context* opt,
                  const rw_beta_params* params, int32_t depth, rw_setup_record* out,
                  int64_t* n_out) {
  int rc;
  if ((rc = need_inputs(ctx, true))) return rc;
  if (!opt || !params || !taus || !out)
    return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep_spec: null argument");
  if (n_setups < 0 || n_slo < 1)
    return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep: bad setup / SLO count");
  if (depth < 1 || depth > 4) return set_err(ctx, RW_ERR_VALIDATION, "rw_sweep_spec: depth must be 1..4");
  if (!(opt->lambda_rps > 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "arrival rate must be positive");
  if (!(opt->kappa > 0.0)) return set_err(ctx, RW_ERR_VALIDATION, "kappa must be positive");
  const int64_t inst = n_setups * (int64_t)n_slo;
  if (n_out) *n_out = inst;
  if (inst == 0) return RW_OK;
  for (int32_t t = 0; t < n_slo; ++t) {
    rw_opt_context o = *opt;
    o.tau_ms = taus[t];
    if ((rc = check_beta_params(ctx, &o, params + t))) return rc;
  }
  if ((rc = validate_profile_index(ctx, pidx, (size_t)n_setups * ctx->m))) return rc;
  CK(cudaSetDevice(ctx->device));
  if ((rc = upload_pidx(ctx, pidx, (size_t)n_setups * ctx->m))) return rc;
  {  // taus + per-SLO params, as rw_sweep_slo_async lays them out
    void* p = ctx->d_setup_ids;
    size_t cap = ctx->setup_ids_cap;
    if ((rc = ensure(ctx, &p, &cap,
                     sizeof(int64_t) * n_setups + (sizeof(double) + sizeof(rw_beta_params)) * n_slo +
                         64)))
      return rc;
    ctx->d_setup_ids = static_cast<int64_t*>(p);
    ctx->setup_ids_cap = cap;
    CK(cudaMemcpyAsync(ctx->d_setup_ids + n_setups, taus, sizeof(double) * n_slo,
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_setup_ids + n_setups + n_slo, params,
                       sizeof(rw_beta_params) * n_slo, cudaMemcpyHostToDevice, ctx->stream));
  }
  // routing_opt.cpp:142-151 bracket per instance (instance k = slo * n_setups + setup)
  std::vector<SpecInst> st(inst);
  for (int64_t k = 0; k < inst; ++k) {
    const rw_beta_params& bp = params[k / n_setups];
    SpecInst& s = st[k];
    s.tau = taus[k / n_setups];
    s.lo = bp.beta_min;
    s.hi = bp.beta_max < 0.0 ? 10.0 / s.tau : bp.beta_max;
    s.eps = bp.epsilon < 0.0 ? (s.hi - s.lo) / 1024.0 : bp.epsilon;
    s.active = s.hi - s.lo > s.eps;
    s.degenerate = !s.active;  // setup_search.cpp:203-208
  }
  std::vector<rw::FracItem> items;
  std::vector<rw::FracRecord> res;
  std::vector<std::vector<int64_t>> node_item(inst);  // per instance: item of tree node
  bool first = true;
  for (;;) {
    items.clear();
    for (int64_t k = 0; k < inst; ++k) {
      SpecInst& s = st[k];
      node_item[k].assign((size_t)1 << depth, -1);
      if (first && s.degenerate) {  // the top penalty, once
        node_item[k][0] = (int64_t)items.size();
        items.push_back({(int32_t)(k % n_setups), (int32_t)(k / n_setups), s.hi});
        continue;
      }
      if (!s.active) continue;
      // breadth-first tree of brackets: node 1 = (lo, hi); children 2n (ok: hi = mid) and
      // 2n + 1 (not ok: lo = mid); a node exists while its bracket is wider than eps
      std::vector<double> nlo((size_t)1 << depth), nhi((size_t)1 << depth);
      nlo[1] = s.lo;
      nhi[1] = s.hi;
      for (size_t nd = 1; nd < ((size_t)1 << depth); ++nd) {
        if (nd > 1 && node_item[k][nd / 2] < 0) continue;  // parent absent
        if (!(nhi[nd] - nlo[nd] > s.eps)) continue;
        const double mid = 0.5 * (nlo[nd] + nhi[nd]);
        node_item[k][nd] = (int64_t)items.size();
        items.push_back({(int32_t)(k % n_setups), (int32_t)(k / n_setups), mid});
        if (2 * nd + 1 < ((size_t)1 << depth)) {
          nlo[2 * nd] = nlo[nd];
          nhi[2 * nd] = mid;
          nlo[2 * nd + 1] = mid;
          nhi[2 * nd + 1] = nhi[nd];
        }
      }
    }
    if (items.empty()) break;
    // one launch: every item is an independent optimize_fractions (persistent CTAs)
    const size_t ni = items.size();
    if ((rc = ensure(ctx, &ctx->d_items, &ctx->items_cap, sizeof(rw::FracItem) * ni))) return rc;
    if ((rc = ensure(ctx, &ctx->d_frac, &ctx->frac_cap, sizeof(rw::FracRecord) * ni))) return rc;
    CK(cudaMemcpyAsync(ctx->d_items, items.data(), sizeof(rw::FracItem) * ni,
                       cudaMemcpyHostToDevice, ctx->stream));
    const int grid = (int)std::min<int64_t>((int64_t)ni, rw::sweep_max_resident(ctx->m, ctx->device));
    if ((rc = ensure_ws(ctx, grid))) return rc;
    rw::Job j = base_job(ctx, rw::JOB_FRAC_BATCH);
    j.prof_idx = ctx->d_prof_idx;
    j.n_items = (int64_t)ni;
    j.taus = reinterpret_cast<const double*>(ctx->d_setup_ids + n_setups);
    j.bps = reinterpret_cast<const rw_beta_params*>(ctx->d_setup_ids + n_setups + n_slo);
    j.opt = *opt;
    j.bp = *params;
    j.frac_items = static_cast<const rw::FracItem*>(ctx->d_items);
    j.frac_out = static_cast<rw::FracRecord*>(ctx->d_frac);
    if ((rc = run(ctx, j, grid))) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    res.resize(ni);
    CK(cudaMemcpy(res.data(), ctx->d_frac, sizeof(rw::FracRecord) * ni, cudaMemcpyDeviceToHost));
    // walk each instance down its realised path (routing_opt.cpp:154-171)
    for (int64_t k = 0; k < inst; ++k) {
      SpecInst& s = st[k];
      for (int64_t it : node_item[k])
        if (it >= 0) s.exec += res[it].exec_passes;
      if (first && s.degenerate) {
        const rw::FracRecord& r = res[node_item[k][0]];
        s.degen = r;
        s.ev += r.eval_passes;
        s.pol += r.polish_passes;
        s.rep += r.repair_calls;
        if (r.status && !s.status) s.status = r.status;
        continue;
      }
      if (!s.active) continue;
      size_t nd = 1;
      while (nd < ((size_t)1 << depth) && node_item[k][nd] >= 0 && s.hi - s.lo > s.eps) {
        const rw::FracRecord& r = res[node_item[k][nd]];
        const double mid = 0.5 * (s.lo + s.hi);
        s.ev += r.eval_passes;
        s.pol += r.polish_passes;
        s.rep += r.repair_calls;
        if (r.status) {
          if (!s.status) s.status = r.status;
          s.active = false;
          break;
        }
        bool in_range = r.out_of_range == 0u;
        bool ok = r.latency_ms <= s.tau && in_range;
        if (s.n_trace == 0 || r.latency_ms < s.tr_best_lat) {  // setup_search.cpp:200-202
          s.tr_best_lat = r.latency_ms;
          s.tr_best_score = r.score;
        }
        s.n_trace++;
        if (ok) {
          s.feasible = true;
          s.beta_star = mid;
          s.best = r;
          s.hi = mid;
          nd = 2 * nd;
        } else {
          s.lo = mid;
          nd = 2 * nd + 1;
        }
      }
      if (!(s.hi - s.lo > s.eps)) s.active = false;
    }
    first = false;
  }
  // records, as evaluate_setup writes them (setup_search.cpp:187-211)
  for (int64_t k = 0; k < inst; ++k) {
    const SpecInst& s = st[k];
    rw_setup_record& r = out[k];
    std::memset(&r, 0, sizeof r);
    r.setup_id = setup_ids ? setup_ids[k % n_setups] : k % n_setups;
    r.status = s.status;
    r.feasible = (!s.status && s.feasible) ? 1 : 0;
    const bool f = s.feasible;
    r.score = f ? s.best.score : (s.n_trace > 0 ? s.tr_best_score : s.degen.score);
    r.latency_ms = f ? s.best.latency_ms : (s.n_trace > 0 ? s.tr_best_lat : s.degen.latency_ms);
    if (s.status) r.score = r.latency_ms = 0.0;
    r.beta = f ? s.beta_star : 0.0;
    r.tau_ms = s.tau;
    for (int i = 0; i < RW_MAX_MODELS; ++i) r.w[i] = (f && i < ctx->m) ? s.best.w[i] : 0.0;
    r.out_of_range = f ? s.best.out_of_range : 0u;
    r.bisect_steps = s.n_trace;
    r.eval_passes = s.ev;
    r.polish_passes = s.pol;
    r.repair_calls = s.rep;
    r.exec_passes = s.exec;
  }
  for (int64_t k = 0; k < inst; ++k)
    if (st[k].status)
      return set_err(ctx, st[k].status,
                     "setup " + std::to_string(out[k].setup_id) + ": solver status " +
                         std::to_string(st[k].status));
  return RW_OK;
}

int rw_sweep_multi(rw_ctx* const* ctxs, int32_t n_ctx, int64_t n_setups,
                   const int64_t* setup_ids, const int32_t* pidx, int32_t n_slo,
                   const double* taus, const rw_opt_context* opt, const rw_beta_params* params,
                   rw_setup_record* out) {
  if (!ctxs || n_ctx < 1 || !ctxs[0])
    return set_err(nullptr, RW_ERR_VALIDATION, "rw_sweep_multi: no contexts");
  for (int r = 0; r < n_ctx; ++r)
    if (!ctxs[r]) return set_err(ctxs[0], RW_ERR_VALIDATION, "rw_sweep_multi: null context");
  if (n_setups < 0 || n_slo < 1)
    return set_err(ctxs[0], RW_ERR_VALIDATION, "rw_sweep: bad setup / SLO count");
  const int64_t inst = n_setups * (int64_t)n_slo;
  std::vector<std::vector<rw_setup_record>> part(n_ctx);
  std::vector<int> rc(n_ctx, RW_OK);
  std::vector<int64_t> got(n_ctx, 0);
  // one host thread drives each GPU (its context owns a stream and device buffers)
  auto shard = [&](int r) {
    const int64_t items = inst > r ? (inst - r + n_ctx - 1) / n_ctx : 0;
    part[r].resize(std::max<int64_t>(items, 1));
    rc[r] = rw_sweep_slo(ctxs[r], n_setups, setup_ids, pidx, n_slo, taus, opt, params, r,
                         n_ctx, part[r].data(), &got[r]);
  };
  if (n_ctx == 1) {
    shard(0);
  } else {
    std::vector<std::thread> pool;
    for (int r = 0; r < n_ctx; ++r) pool.emplace_back(shard, r);
    for (auto& t : pool) t.join();
  }
  for (int r = 0; r < n_ctx; ++r)
    if (rc[r] != RW_OK) {
      if (r != 0) ctxs[0]->err = "shard " + std::to_string(r) + ": " + ctxs[r]->err;
      return rc[r];
    }
  // the combine: interleaved shards back into instance order
  for (int r = 0; r < n_ctx; ++r)
    for (int64_t i = 0; i < got[r]; ++i) out[r + i * n_ctx] = part[r][i];
  return RW_OK;
}

int rw_sweep(rw_ctx* ctx, int64_t n_setups, const int64_t* setup_ids, const int32_t* pidx,
             const rw_opt_context* opt, const rw_beta_params* params, int32_t shard_rank,
             int32_t shard_count, rw_setup_record* out, int64_t* n_out) {
  int rc = rw_sweep_async(ctx, n_setups, setup_ids, pidx, opt, params, shard_rank, shard_count);
  if (rc) return rc;
  return rw_sweep_fetch(ctx, out, n_out);
}

}  // extern "C"
