// zp_fast_p59.cu -- fast-path instantiation for p = 59 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(59)
