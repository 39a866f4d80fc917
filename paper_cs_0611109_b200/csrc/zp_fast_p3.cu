// zp_fast_p3.cu -- fast-path instantiation for p = 3 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST(3)
