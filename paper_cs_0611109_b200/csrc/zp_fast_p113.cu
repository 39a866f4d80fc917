// zp_fast_p113.cu -- fast-path instantiation for p = 113 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(113)
