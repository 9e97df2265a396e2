// Microbenchmark (diagnostics, not product): streaming an L2-resident N x 4 f64 matrix
// with different lane->row mappings, to size the pass kernel's load layout.
//   A: lane = row, two LDG.128 per row (current producer layout)
//   B: lane pair = row, one LDG.128 per lane (512 contiguous bytes per instruction)
//   C: like A but each CTA streams its own copy offset (no L1 sharing effects)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_l2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) kA(const double* __restrict__ s, int n, int reps, double* out) {
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    for (int base = 0; base < n; base += 256 * 8) {
      double v[8][4];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        int j = min(base + g * 256 + (int)threadIdx.x, n - 1);
        const double2* p = reinterpret_cast<const double2*>(s + (size_t)j * 4);
        double2 x = __ldg(p), y = __ldg(p + 1);
        v[g][0] = x.x; v[g][1] = x.y; v[g][2] = y.x; v[g][3] = y.y;
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        double b = v[g][0];
#pragma unroll
        for (int i = 1; i < 4; ++i) b = b < v[g][i] ? v[g][i] : b;
        acc += b;
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(256) kB(const double* __restrict__ s, int n, int reps, double* out) {
  double acc = 0.0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* s2 = reinterpret_cast<const double2*>(s);
  const int n2 = n * 2;  // double2 count
  for (int r = 0; r < reps; ++r) {
    for (int base = 0; base < n2; base += 256 * 8) {
      double2 v[8];
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        int q = min(base + (w * 8 + g) * 32 + lane, n2 - 1);
        v[g] = __ldg(s2 + q);
      }
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        double b = v[g].x < v[g].y ? v[g].y : v[g].x;
        double o = __shfl_xor_sync(0xffffffffu, b, 1);
        b = b < o ? o : b;
        acc += b;
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int n = 100000;
  double* d;
  double* o;
  cudaMalloc(&d, sizeof(double) * n * 4);
  cudaMalloc(&o, 64);
  cudaMemset(d, 0, sizeof(double) * n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int reps = 20;
  for (int grid : {1, 148, 296, 444, 592}) {
    for (int kind = 0; kind < 2; ++kind) {
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(e0);
        if (kind == 0) kA<<<grid, 256>>>(d, n, reps, o);
        else kB<<<grid, 256>>>(d, n, reps, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)grid * reps * n * 32.0;
      printf("kernel %c grid %4d: %.3f ms  %.1f GB/s  per-CTA pass %.1f us\n", kind ? 'B' : 'A', grid,
             ms, bytes / ms / 1e6, ms * 1e3 / reps);
    }
  }
  return 0;
}
