// zp_fast_p241.cu -- fast-path instantiation for p = 241 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(241)
