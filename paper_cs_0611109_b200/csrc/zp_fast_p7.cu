// zp_fast_p7.cu -- fast-path instantiation for p = 7 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST(7)
