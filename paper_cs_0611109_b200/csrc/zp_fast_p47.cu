// zp_fast_p47.cu -- fast-path instantiation for p = 47 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(47)
