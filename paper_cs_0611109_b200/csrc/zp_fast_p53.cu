// zp_fast_p53.cu -- fast-path instantiation for p = 53 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(53)
