// zp_generic_b.cu -- explicit instantiations of the generic kernel (zp_generic.cuh), split over
// three translation units so that the build compiles them in parallel.
#include "zp_generic.cuh"

namespace zp {
namespace gen {
template cudaError_t launch_p<7>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<67>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<83>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<127>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<149>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<163>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<179>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<197>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<223>(const ZpArgs&, int, cudaStream_t, int);
template cudaError_t launch_p<239>(const ZpArgs&, int, cudaStream_t, int);
}  // namespace gen
}  // namespace zp
