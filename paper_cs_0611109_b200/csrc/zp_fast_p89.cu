// zp_fast_p89.cu -- fast-path instantiation for p = 89 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(89)
