// zp_fast_p31.cu -- fast-path instantiation for p = 31 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST(31)
