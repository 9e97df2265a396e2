// rw_kernels.cu — dispatch from the runtime model count to the compiled instantiations.
//
// Template choice: MM = model-count bucket (register tile width for a row), L = rows per
// thread per tile, T = threads per CTA.  One CTA = one setup at a time (persistent).
// Each bucket is instantiated in its own translation unit (rw_inst_m*.cu) so the build
// parallelises.
#include <cuda_runtime.h>

#include "rw_job.h"

namespace rw {

#define RW_DECLARE(MM)                                          \
  int launch_m##MM(const Job& job, int grid, cudaStream_t st); \
  int resident_m##MM(int device);
RW_DECLARE(4)
RW_DECLARE(8)
RW_DECLARE(16)
RW_DECLARE(32)
#undef RW_DECLARE

int launch_job(const Job& job, int grid, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (job.m <= 4) return launch_m4(job, grid, st);
  if (job.m <= 8) return launch_m8(job, grid, st);
  if (job.m <= 16) return launch_m16(job, grid, st);
  return launch_m32(job, grid, st);
}

int sweep_max_resident(int m, int device) {
  if (m <= 4) return resident_m4(device);
  if (m <= 8) return resident_m8(device);
  if (m <= 16) return resident_m16(device);
  return resident_m32(device);
}

}  // namespace rw
