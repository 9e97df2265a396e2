#include "rw_inst.cuh"
RW_INSTANTIATE(32, 8, 256)
