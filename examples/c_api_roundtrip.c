/*
 * c_api_roundtrip.c -- the C ABI of libraid6c.so used from plain C (no Python, no PyTorch):
 * encode a batch of stripes, erase a pair of strips in every stripe (all classes: DD, DP, DQ, PQ),
 * rebuild them, and check the result byte for byte against the original (include/raid6c.h).
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_roundtrip.c \
 *       -L paper_cs_0611109_b200 -lraid6c -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,paper_cs_0611109_b200 -o c_api_roundtrip
 *   ./c_api_roundtrip [p] [N] [bytes] [stripes]      (defaults: 13 12 1000003 8)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "raid6c.h"

#define CHECK_R(call)                                                                       \
  do {                                                                                      \
    raid6c_status s_ = (call);                                                              \
    if (s_ != RAID6C_OK) {                                                                  \
      fprintf(stderr, "%s:%d %s -> %s %s\n", __FILE__, __LINE__, #call,                     \
              raid6c_status_string(s_), raid6c_last_cuda_error());                          \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)
#define CHECK_C(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

static uint64_t splitmix(uint64_t* x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  const int p = argc > 1 ? atoi(argv[1]) : 13;
  const int N = argc > 2 ? atoi(argv[2]) : 12;
  const size_t bytes = argc > 3 ? (size_t)atoll(argv[3]) : 1000003;
  const int S = argc > 4 ? atoi(argv[4]) : 8;
  const size_t pb = raid6c_parity_bytes(p, bytes);
  if (pb == 0) {
    fprintf(stderr, "invalid p = %d\n", p);
    return 1;
  }
  const size_t ss = (bytes + 255) / 256 * 256, ps = (pb + 255) / 256 * 256;
  const size_t data_sz = (size_t)S * N * ss, par_sz = (size_t)S * 2 * ps;

  uint8_t *h_data = malloc(data_sz), *h_par = malloc(par_sz), *h_chk = malloc(data_sz > par_sz ? data_sz : par_sz);
  uint64_t seed = 42;
  for (size_t i = 0; i < data_sz; i++) h_data[i] = (uint8_t)splitmix(&seed);
  uint8_t *d_data, *d_par;
  CHECK_C(cudaMalloc((void**)&d_data, data_sz));
  CHECK_C(cudaMalloc((void**)&d_par, par_sz));
  CHECK_C(cudaMemcpy(d_data, h_data, data_sz, cudaMemcpyHostToDevice));
  CHECK_C(cudaMemset(d_par, 0, par_sz));

  raid6c_plan plan;
  CHECK_R(raid6c_plan_create(&plan, p, N, bytes, 0, NULL));
  CHECK_R(raid6c_encode_strided(plan, d_data, ss, (size_t)N * ss, d_par, d_par + ps, 2 * ps, S));
  CHECK_R(raid6c_sync(plan));
  CHECK_C(cudaMemcpy(h_par, d_par, par_sz, cudaMemcpyDeviceToHost));

  /* one erasure pair per stripe, cycling through the classes DD, DP, DQ, PQ */
  raid6c_erasure* er = malloc(sizeof(raid6c_erasure) * S);
  for (int s = 0; s < S; s++) {
    const int cls = s % 4, a = (3 * s + 1) % N, b = (5 * s + 2) % N;
    if (cls == 0) { er[s].lost_i = a; er[s].lost_j = (a == b) ? (a + 1) % N : b; }
    if (cls == 1) { er[s].lost_i = N; er[s].lost_j = a; }   /* (P, d_a): either order */
    if (cls == 2) { er[s].lost_i = a; er[s].lost_j = N + 1; }
    if (cls == 3) { er[s].lost_i = N; er[s].lost_j = N + 1; }
    if (N == 1 && cls == 0) { er[s].lost_i = 0; er[s].lost_j = N; }
    for (int t = 0; t < 2; t++) {  /* poison the lost strips: they are outputs only */
      const int k = t ? er[s].lost_j : er[s].lost_i;
      uint8_t* dst = k < N ? d_data + (size_t)s * N * ss + (size_t)k * ss : d_par + (size_t)s * 2 * ps + (size_t)(k - N) * ps;
      CHECK_C(cudaMemset(dst, 0xA5, k < N ? bytes : pb));
    }
  }
  CHECK_R(raid6c_recover_strided(plan, d_data, ss, (size_t)N * ss, d_par, d_par + ps, 2 * ps, S, er, S, 0));
  CHECK_R(raid6c_sync(plan));

  size_t bad = 0;
  CHECK_C(cudaMemcpy(h_chk, d_data, data_sz, cudaMemcpyDeviceToHost));
  for (int s = 0; s < S; s++)
    for (int k = 0; k < N; k++)
      bad += memcmp(h_chk + (size_t)s * N * ss + (size_t)k * ss, h_data + (size_t)s * N * ss + (size_t)k * ss, bytes) != 0;
  CHECK_C(cudaMemcpy(h_chk, d_par, par_sz, cudaMemcpyDeviceToHost));
  for (int s = 0; s < S; s++)
    for (int k = 0; k < 2; k++)
      bad += memcmp(h_chk + (size_t)s * 2 * ps + (size_t)k * ps, h_par + (size_t)s * 2 * ps + (size_t)k * ps, pb) != 0;

  /* a single lost strip: lost_j = RAID6C_NONE (runs as the pair (lost_i, Q): d_0 of stripe 0 is
   * rebuilt from the other strips and P, and the intact Q is regenerated with it) */
  CHECK_C(cudaMemset(d_data, 0xA5, bytes));
  raid6c_erasure one = {0, RAID6C_NONE};
  CHECK_R(raid6c_recover_strided(plan, d_data, ss, (size_t)N * ss, d_par, d_par + ps, 2 * ps, 1, &one, 1, 0));
  CHECK_R(raid6c_sync(plan));
  CHECK_C(cudaMemcpy(h_chk, d_data, bytes, cudaMemcpyDeviceToHost));
  bad += memcmp(h_chk, h_data, bytes) != 0;
  CHECK_C(cudaMemcpy(h_chk, d_par + ps, pb, cudaMemcpyDeviceToHost));
  bad += memcmp(h_chk, h_par + ps, pb) != 0;

  /* an argument error is synchronous and has no side effect */
  raid6c_erasure badpair = {0, 0};
  const raid6c_status e = raid6c_recover_strided(plan, d_data, ss, (size_t)N * ss, d_par, d_par + ps, 2 * ps, 1,
                                                 &badpair, 1, 0);
  CHECK_R(raid6c_plan_destroy(plan));
  cudaFree(d_data);
  cudaFree(d_par);
  free(h_data); free(h_par); free(h_chk); free(er);
  printf("p=%d N=%d bytes=%zu stripes=%d: %zu strips differ after recovery; bad-pair status: %s\n", p, N, bytes, S,
         bad, raid6c_status_string(e));
  return (bad == 0 && e == RAID6C_E_INVALID_INDEX) ? 0 : 1;
}
