#include "rw_inst.cuh"
#ifndef RW_L4
#define RW_L4 16  // rows per warp block / 32 (experiments: -DRW_L4=8, 32)
#endif
RW_INSTANTIATE(4, RW_L4, 256)
