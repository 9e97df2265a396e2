#include "rw_inst.cuh"
RW_INSTANTIATE(4, 16, 256)
