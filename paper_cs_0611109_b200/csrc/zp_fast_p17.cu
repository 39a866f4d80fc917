// zp_fast_p17.cu -- fast-path instantiation for p = 17 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(17)
