// zp_fast_p233.cu -- fast-path instantiation for p = 233 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(233)
