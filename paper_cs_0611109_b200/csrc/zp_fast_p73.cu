// zp_fast_p73.cu -- fast-path instantiation for p = 73 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST(73)
