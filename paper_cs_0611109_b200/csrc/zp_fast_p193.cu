// zp_fast_p193.cu -- fast-path instantiation for p = 193 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(193)
