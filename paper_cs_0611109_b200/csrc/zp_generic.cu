// zp_generic.cu -- dispatch of the generic kernel (zp_generic.cuh) by p; the instantiations
// live in zp_generic_{a,b,c}.cu.
#include "zp_generic.cuh"

namespace zp {
namespace gen {
extern template cudaError_t launch_p<3>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<7>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<31>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<73>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<67>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<71>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<79>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<83>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<103>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<107>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<127>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<131>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<139>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<149>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<151>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<157>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<163>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<167>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<173>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<179>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<181>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<191>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<197>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<199>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<211>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<223>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<227>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<229>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<239>(const ZpArgs&, int, cudaStream_t, int);
extern template cudaError_t launch_p<251>(const ZpArgs&, int, cudaStream_t, int);
}  // namespace gen

// The 26 primes whose period lcm(p-1, 32) exceeds 32 lanes, plus the fast primes without
// extended-code kernels (3, 7, 31, 73: Theorem 25.3 fails, so never reached by a valid plan).
cudaError_t generic_launch(const ZpArgs& a, int p, int mode, cudaStream_t st, int num_sms) {
  switch (p) {
#define ZP_GEN_CASE(PP) \
  case PP: return gen::launch_p<PP>(a, mode, st, num_sms);
    ZP_GEN_CASE(3) ZP_GEN_CASE(7) ZP_GEN_CASE(31) ZP_GEN_CASE(73)
    ZP_GEN_CASE(67) ZP_GEN_CASE(71) ZP_GEN_CASE(79) ZP_GEN_CASE(83) ZP_GEN_CASE(103) ZP_GEN_CASE(107)
    ZP_GEN_CASE(127) ZP_GEN_CASE(131) ZP_GEN_CASE(139) ZP_GEN_CASE(149) ZP_GEN_CASE(151) ZP_GEN_CASE(157)
    ZP_GEN_CASE(163) ZP_GEN_CASE(167) ZP_GEN_CASE(173) ZP_GEN_CASE(179) ZP_GEN_CASE(181) ZP_GEN_CASE(191)
    ZP_GEN_CASE(197) ZP_GEN_CASE(199) ZP_GEN_CASE(211) ZP_GEN_CASE(223) ZP_GEN_CASE(227) ZP_GEN_CASE(229)
    ZP_GEN_CASE(239) ZP_GEN_CASE(251)
#undef ZP_GEN_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace zp
