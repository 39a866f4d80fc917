// zp_generic_c.cu -- explicit instantiations of the generic kernel (zp_generic.cuh), split over
// three translation units so that the build compiles them in parallel.
#include "zp_generic.cuh"

namespace zp {
namespace gen {
template cudaError_t launch_p<31>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<71>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<103>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<131>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<151>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<167>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<181>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<199>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<227>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<251>(const ZpArgs&, int, cudaStream_t, int);
}  // namespace gen
}  // namespace zp
