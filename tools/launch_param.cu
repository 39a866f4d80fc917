// Launch cost of a 6.3 KB __grid_constant__ parameter block (ZpArgs-sized) vs a 64-byte one,
// for 8-CTA launches, from a CUDA graph and from a stream (tools/README.md).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
struct Big { const uint8_t* p[780]; int64_t x[8]; };   // ~6.3 KB
struct Small { const uint8_t* p[6]; int64_t x[2]; };
__global__ void kbig(const __grid_constant__ Big a) { if (a.x[0] == 12345) printf("x"); }
__global__ void ksmall(const __grid_constant__ Small a) { if (a.x[0] == 12345) printf("x"); }
int main() {
  printf("sizeof Big %zu\n", sizeof(Big));
  cudaStream_t s; cudaStreamCreate(&s);
  Big b = {}; Small sm = {};
  for (int v = 0; v < 2; v++) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 16; i++) { if (v == 0) kbig<<<8, 288, 0, s>>>(b); else ksmall<<<8, 288, 0, s>>>(sm); }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 5; i++) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 100; i++) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: %.2f us per launch (graph)\n", v == 0 ? "6.3KB param" : "64B param", 1e3 * ms / 1600);
    // plain stream launches back to back
    cudaEventRecord(e0, s);
    for (int i = 0; i < 1600; i++) { if (v == 0) kbig<<<8, 288, 0, s>>>(b); else ksmall<<<8, 288, 0, s>>>(sm); }
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: %.2f us per launch (stream)\n", v == 0 ? "6.3KB param" : "64B param", 1e3 * ms / 1600);
  }
  return 0;
}
