#include "rw_inst.cuh"
RW_INSTANTIATE(8, 8, 512)
