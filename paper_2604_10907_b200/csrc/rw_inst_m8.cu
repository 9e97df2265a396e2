#include "rw_inst.cuh"
#ifndef RW_L8
#define RW_L8 16  // rows per warp block / 32 (experiment: -DRW_L8=8)
#endif
RW_INSTANTIATE(8, RW_L8, 256)
