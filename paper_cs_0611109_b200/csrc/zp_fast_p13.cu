// zp_fast_p13.cu -- fast-path instantiation for p = 13 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(13)
