// zp_fast_p97.cu -- fast-path instantiation for p = 97 (see zp_fast.cuh).
#include "zp_fast.cuh"
ZP_INSTANTIATE_FAST_EXT(97)
