// zp_fast_p11.cu -- fast-path instantiation for p = 11 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(11)
