// zp_fast_p37.cu -- fast-path instantiation for p = 37 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(37)
