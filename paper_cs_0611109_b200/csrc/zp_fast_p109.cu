// zp_fast_p109.cu -- fast-path instantiation for p = 109 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(109)
