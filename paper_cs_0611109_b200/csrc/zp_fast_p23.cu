// zp_fast_p23.cu -- fast-path instantiation for p = 23 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(23)
