#include "rw_inst.cuh"
RW_INSTANTIATE(16, 16, 256)
