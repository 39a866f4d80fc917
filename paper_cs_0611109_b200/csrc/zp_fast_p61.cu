// zp_fast_p61.cu -- fast-path instantiation for p = 61 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(61)
