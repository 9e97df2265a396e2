// One instantiation of the solver kernel + its launcher (included by rw_inst_m*.cu).
#pragma once
#include <cuda_runtime.h>

#include "rw_job.h"
#include "rw_solver.cuh"

#define RW_INSTANTIATE(MM, L, T)                                                              \
  namespace rw {                                                                              \
  int launch_m##MM(const Job& job, int grid, cudaStream_t st) {                               \
    using SM = Smem<MM, L, T>;                                                                \
    /* the smem opt-in is per device: remember it per device ordinal */                      \
    static bool configured[64] = {};                                                          \
    int dev = 0;                                                                              \
    cudaGetDevice(&dev);                                                                      \
    if (dev < 0 || dev >= 64 || !configured[dev]) {                                           \
      cudaError_t e = cudaFuncSetAttribute(solver_kernel<MM, L, T>,                          \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                           (int)sizeof(SM));                                  \
      if (e != cudaSuccess) return (int)e;                                                    \
      if (dev >= 0 && dev < 64) configured[dev] = true;                                       \
    }                                                                                         \
    solver_kernel<MM, L, T><<<grid, T, sizeof(SM), st>>>(job);                                \
    return (int)cudaGetLastError();                                                           \
  }                                                                                           \
  int resident_m##MM(int device) {                                                            \
    using SM = Smem<MM, L, T>;                                                                \
    cudaFuncSetAttribute(solver_kernel<MM, L, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)sizeof(SM));                                                    \
    int per_sm = 0;                                                                           \
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solver_kernel<MM, L, T>, T,   \
                                                      sizeof(SM)) != cudaSuccess)             \
      per_sm = 1;                                                                             \
    int sms = 0;                                                                              \
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);                    \
    return (per_sm < 1 ? 1 : per_sm) * sms;                                                   \
  }                                                                                           \
  }
