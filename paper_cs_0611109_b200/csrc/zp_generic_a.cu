// zp_generic_a.cu -- explicit instantiations of the generic kernel (zp_generic.cuh), split over
// three translation units so that the build compiles them in parallel.
#include "zp_generic.cuh"

namespace zp {
namespace gen {
template cudaError_t launch_p<3>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<73>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<79>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<107>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<139>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<157>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<173>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<191>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<211>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<229>(const ZpArgs&, int, cudaStream_t, int);
}  // namespace gen
}  // namespace zp
