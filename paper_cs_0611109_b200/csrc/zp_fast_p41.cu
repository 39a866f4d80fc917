// zp_fast_p41.cu -- fast-path instantiation for p = 41 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(41)
