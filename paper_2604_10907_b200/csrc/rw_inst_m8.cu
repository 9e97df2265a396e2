#include "rw_inst.cuh"
RW_INSTANTIATE(8, 16, 256)
