// zp_fast_p5.cu -- fast-path instantiation for p = 5 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(5)
