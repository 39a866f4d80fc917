// zp_fast_p101.cu -- fast-path instantiation for p = 101 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(101)
