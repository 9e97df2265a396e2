// Microbenchmark (diagnostics, not product): per-warp TMA rings vs CTA-wide stages for the
// eval pass's stream of a 1M x 8 f64 L2-resident matrix, WITH the pass's per-row work
// (priced argmax over 8 models, binade quanta, sums, packed counts) so the numbers bound
// what produce() can reach.
//   A: per-warp ring, S slots of SR rows, one 1-D bulk copy per warp stage (current).
//   B: CTA-wide stage of WP*SR rows in ONE bulk copy, S slots; each warp consumes its
//      SR-row part; the last warp to finish a stage refills its slot (no empty barrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbs tools/microbench_stage.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void load(void* dst, const void* src, unsigned bytes,
                                     unsigned long long* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(b),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

struct Acc {
  long long Q = 0;
  double sb = 0.0, sa = 0.0;
  unsigned long long pk[2] = {0, 0};
  bool tie = false;
};
// the pass's per-row work on one 8-model row read from smem (row-major, 64 B)
__device__ __forceinline__ void row_work(const double* v, const double (&a)[8], double scale,
                                         Acc& acc) {
  double bj = v[0] - a[0];
  int arg = 0;
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    const double x = v[i] - a[i];
    const bool gt = x > bj;
    bj = gt ? x : bj;
    arg = gt ? i : arg;
  }
  const double y = fabs(bj) * scale;
  const double t = y + 0x1p52;
  const long long q = __double_as_longlong(t) - 0x4330000000000000ll;
  acc.tie |= (fabs((t - 0x1p52) - y) == 0.5);
  acc.Q += (bj < 0.0) ? -q : q;
  acc.sb += bj;
  acc.sa += fabs(bj);
  acc.pk[arg >> 2] += 1ull << ((arg & 3) * 16);
}

template <int MODE>
__global__ void stream(const double* __restrict__ s, int n, int passes, int S, int SR,
                       double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int W = blockDim.x / 32, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = 8, row_bytes = 64;
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.01 * i;
  Acc acc;
  const double scale = 0x1p40;
  if (MODE == 0) {  // per-warp rings
    const int stage_bytes = SR * row_bytes;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + (size_t)W * S * stage_bytes);
    if (lane == 0)
      for (int q = 0; q < S; ++q) mbar_init(&bars[w * S + q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    unsigned char* ring = sm + (size_t)w * S * stage_bytes;
    const int per_pass = (n + W * SR - 1) / (W * SR);
    const long long total = (long long)per_pass * passes;
    auto issue = [&](long long k) {
      if (lane == 0 && k < total) {
        const int t = (int)(k % per_pass);
        const int r0 = min((t * W + w) * SR, n - SR);
        load(ring + (k % S) * stage_bytes, s + (size_t)r0 * m, (unsigned)stage_bytes,
             &bars[w * S + (k % S)]);
      }
    };
    for (int k = 0; k < S - 1; ++k) issue(k);
    for (long long k = 0; k < total; ++k) {
      issue(k + S - 1);
      mbar_wait(&bars[w * S + (k % S)], (unsigned)((k / S) & 1));
      const double* st = reinterpret_cast<const double*>(ring + (k % S) * stage_bytes);
      for (int r = lane; r < SR; r += 32) row_work(st + r * m, a, scale, acc);
      __syncwarp();
    }
  } else {  // CTA-wide stages, last finisher refills
    const int WP = W;
    const int stage_bytes = WP * SR * row_bytes;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + (size_t)S * stage_bytes);
    int* done = reinterpret_cast<int*>(bars + S);
    if (threadIdx.x == 0) {
      for (int q = 0; q < S; ++q) {
        mbar_init(&bars[q], 1);
        done[q] = 0;
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int per_pass = (n + WP * SR - 1) / (WP * SR);
    const long long total = (long long)per_pass * passes;
    auto issue = [&](long long k) {
      if (k < total) {
        const int t = (int)(k % per_pass);
        const int r0 = min(t * WP * SR, n - WP * SR);
        load(sm + (k % S) * stage_bytes, s + (size_t)r0 * m, (unsigned)stage_bytes,
             &bars[k % S]);
      }
    };
    if (threadIdx.x == 0)
      for (int k = 0; k < S; ++k) issue(k);
    for (long long k = 0; k < total; ++k) {
      mbar_wait(&bars[k % S], (unsigned)((k / S) & 1));
      const double* st =
          reinterpret_cast<const double*>(sm + (k % S) * stage_bytes + (size_t)w * SR * row_bytes);
      for (int r = lane; r < SR; r += 32) row_work(st + r * m, a, scale, acc);
      __syncwarp();
      if (lane == 0) {
        if (atomicAdd(&done[k % S], 1) == WP - 1) {  // last warp out refills the slot
          done[k % S] = 0;
          issue(k + S);
        }
      }
    }
  }
  if (acc.sb == 1234.5 && acc.Q == 7 && acc.pk[0] == 3 && acc.tie) out[0] = acc.sa;
}

int main() {
  const int n = 1 << 20, passes = 6;
  double* d;
  cudaMalloc(&d, (size_t)n * 8 * 8);
  cudaMemset(d, 0, (size_t)n * 8 * 8);
  double* o;
  cudaMalloc(&o, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg { int mode, ctas, warps, S, SR; };
  Cfg cfgs[] = {{0, 2, 7, 2, 64},  {0, 2, 7, 2, 128}, {0, 2, 8, 2, 64},  {1, 2, 7, 2, 64},
                {1, 2, 7, 3, 64},  {1, 2, 8, 2, 64},  {1, 2, 8, 3, 64},  {1, 2, 7, 2, 128},
                {1, 1, 15, 3, 64}, {1, 1, 16, 3, 64}, {1, 2, 8, 4, 32},  {1, 2, 7, 4, 32}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Cfg& c : cfgs) {
    const size_t smem = (c.mode == 0 ? (size_t)c.warps : 1) * c.S *
                            (c.mode == 0 ? c.SR * 64 : (size_t)c.warps * c.SR * 64) +
                        64 * c.S + 64 * c.warps;
    if (smem > 227 * 1024 || smem * c.ctas > 228 * 1024) {
      printf("skip mode %d %d/%d/%d/%d (smem %zu)\n", c.mode, c.ctas, c.warps, c.S, c.SR, smem);
      continue;
    }
    const int grid = sms * c.ctas;
    auto run = [&](int p) {
      if (c.mode == 0) stream<0><<<grid, c.warps * 32, smem>>>(d, n, p, c.S, c.SR, o);
      else stream<1><<<grid, c.warps * 32, smem>>>(d, n, p, c.S, c.SR, o);
    };
    run(1);
    cudaEventRecord(e0);
    run(passes);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * passes * n * 64;
    printf("mode %s ctas/SM %d warps %2d slots %d rows/warp-stage %3d op %6d B: %8.1f GB/s  "
           "%.3e rows/s (%s)\n",
           c.mode ? "CTA-stage" : "warp-ring", c.ctas, c.warps, c.S, c.SR,
           c.mode ? c.warps * c.SR * 64 : c.SR * 64, bytes / ms / 1e6,
           (double)grid * passes * n / (ms / 1e3), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
