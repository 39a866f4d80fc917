// zp_fast_p43.cu -- fast-path instantiation for p = 43 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(43)
