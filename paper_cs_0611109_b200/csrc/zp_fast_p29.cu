// zp_fast_p29.cu -- fast-path instantiation for p = 29 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(29)
