// zp_fast_p19.cu -- fast-path instantiation for p = 19 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(19)
