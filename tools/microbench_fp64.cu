// Microbenchmark (diagnostics): the B200's FP64 issue rate (SURVEY.md H7 — the roof the
// pass's compare/quanta chains would hit once the stream stops bounding it).  DADD, DFMA
// and DSETP+select chains, 8 independent chains per thread, all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbf tools/microbench_fp64.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __dadd_rn(x[i], a);
      else if (OP == 1) x[i] = __fma_rn(x[i], a, b);
      else x[i] = (x[i] > b) ? x[i] - a : x[i] + a;  // DSETP + DADD + select
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 14, threads = 512, blocks = sms * 4;
  const char* names[] = {"DADD", "DFMA", "DSETP+DADD+SEL"};
  for (int op = 0; op < 3; ++op) {
    auto launch = [&] {
      if (op == 0) k<0><<<blocks, threads>>>(o, iters, 1e-300, 0.5);
      else if (op == 1) k<1><<<blocks, threads>>>(o, iters, 0.999999, 1e-9);
      else k<2><<<blocks, threads>>>(o, iters, 1e-300, 0.5);
    };
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    printf("%-16s %8.2f Gop/s = %6.1f ops/clk/SM at 1.965 GHz (%s)\n", names[op], ops / ms / 1e6,
           ops / (ms / 1e3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
