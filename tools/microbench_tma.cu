// Microbenchmark (diagnostics, not product): how fast can CTAs stream an L2-resident
// 1M x 8 f64 score matrix (C3, 64 MB) with per-warp 1-D bulk-copy (TMA) rings, as a
// function of bytes in flight — sizes the eval pass's ring (rw_solver.cuh produce()).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbt tools/microbench_tma.cu
//   ./mbt   -> one line per (CTAs/SM, warps, slots, stage bytes): aggregate GB/s
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
__device__ __forceinline__ void load_stage(void* dst, const void* src, unsigned bytes,
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

// Each warp streams stages (rows [(t*W + w)*SR, +SR)) of the whole matrix `passes` times
// through an S-slot ring; the consumer reads every double of the stage (LDS) like a pass.
__global__ void stream(const double* __restrict__ s, int n, int m, int passes, int S, int SR,
                       double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int W = blockDim.x / 32, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stage_bytes = SR * m * 8;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + (size_t)W * S * stage_bytes);
  if (lane == 0)
    for (int q = 0; q < S; ++q) mbar_init(&bars[w * S + q], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned char* ring = sm + (size_t)w * S * stage_bytes;
  const int per_pass = (n + W * SR - 1) / (W * SR);
  const long long total = (long long)per_pass * passes;
  // stage k of this warp: pass k / per_pass, stage index k % per_pass
  auto issue = [&](long long k) {
    if (lane == 0 && k < total) {
      const int t = (int)(k % per_pass);
      const int r0 = (t * W + w) * SR;
      if (r0 < n) {
        const int nv = min(SR, n - r0);
        load_stage(ring + (k % S) * stage_bytes, s + (size_t)r0 * m, (unsigned)(nv * m * 8),
                   &bars[w * S + (k % S)]);
      } else {  // keep the phase sequence: arrive on an empty stage
        unsigned b = (unsigned)__cvta_generic_to_shared(&bars[w * S + (k % S)]);
        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(b)
                     : "memory");
      }
    }
  };
  for (int k = 0; k < S - 1; ++k) issue(k);
  double acc = 0.0;
  for (long long k = 0; k < total; ++k) {
    issue(k + S - 1);
    mbar_wait(&bars[w * S + (k % S)], (unsigned)((k / S) & 1));
    const double* st = reinterpret_cast<const double*>(ring + (k % S) * stage_bytes);
    for (int e = lane; e < SR * m; e += 32) acc += st[e];
    __syncwarp();
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const int n = 1 << 20, m = 8, passes = 6;
  double* d;
  cudaMalloc(&d, (size_t)n * m * 8);
  cudaMemset(d, 0, (size_t)n * m * 8);
  double* o;
  cudaMalloc(&o, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Cfg { int ctas_per_sm, warps, S, SR; };
  Cfg cfgs[] = {{2, 7, 2, 64}, {2, 7, 3, 64}, {2, 7, 4, 64}, {2, 8, 3, 64}, {2, 7, 2, 128},
                {2, 7, 3, 128}, {1, 8, 4, 128}, {1, 14, 3, 64}, {1, 16, 4, 64}, {1, 8, 6, 128},
                {1, 8, 3, 256}, {2, 4, 4, 128}, {1, 16, 6, 32}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Cfg& c : cfgs) {
    const size_t smem = (size_t)c.warps * c.S * c.SR * m * 8 + (size_t)c.warps * c.S * 8;
    if (smem > 227 * 1024 || smem * c.ctas_per_sm > 228 * 1024) {
      printf("skip %d/%d/%d/%d (smem %zu)\n", c.ctas_per_sm, c.warps, c.S, c.SR, smem);
      continue;
    }
    const int grid = sms * c.ctas_per_sm;
    stream<<<grid, c.warps * 32, smem>>>(d, n, m, 1, c.S, c.SR, o);
    cudaEventRecord(e0);
    stream<<<grid, c.warps * 32, smem>>>(d, n, m, passes, c.S, c.SR, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * passes * n * m * 8;
    printf("ctas/SM %d warps %2d slots %d stage %5d B  in-flight/SM %6zu B : %8.1f GB/s  (%s)\n",
           c.ctas_per_sm, c.warps, c.S, c.SR * m * 8,
           (size_t)c.ctas_per_sm * c.warps * (c.S - 1) * c.SR * m * 8, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
