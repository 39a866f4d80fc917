// zp_fast_p257.cu -- fast-path instantiation for p = 257 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(257)
