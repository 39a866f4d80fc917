// zp_fast_p137.cu -- fast-path instantiation for p = 137 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(137)
