// zp_args.h -- launch descriptor shared by the host side of libraid6c and its kernels.
// (Product code only; nothing here is shared with oracle/.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "raid6c.h"

namespace zp {

// Extended code (NEXT-2, N > p): per-stripe multiplier u for the DP / DD solves, a ring element
// of R_p given by the exponents of its nonzero coefficients (u = sum_i x^{e_i}), computed on the
// host: u = g_j^{-1} (DP) or (g_x + g_y)^{-1} (DD), g_k the Eq. (qext) coefficient of disk k.
struct ExtProg {
  int32_t nu;
  // geo_bz != 0: u = x^{geo_e0} (1 + x^z)^{-1} with geo_bz = 2z mod p (the pair's coefficients
  // are both monomials or both binomials 1 + x^c): evaluated as the basic code's geometric series
  int16_t geo_bz, geo_e0;
  uint16_t e[RAID6C_MAX_P - 1];
};

// One launch = a batch of stripes with a common (p, N, bytes).  Strip k of stripe s lives
// at base[k] + s * (k < N ? data_stride : parity_stride).
struct ZpArgs {
  const uint8_t* base[RAID6C_MAX_STRIPS];
  uint64_t data_stride;
  uint64_t parity_stride;
  uint64_t bytes;   // data strip length
  uint64_t pbytes;  // parity strip length (W*n bits rounded up to bytes)
  int N;
  int num_stripes;
  // Erasure pair per stripe: er[s] if er != nullptr, else (ei, ej).  Encode = (N, N+1).
  const int2* er;
  int er_stride;  // er[s * er_stride] (0 = one pair for every stripe)
  int ei, ej;
  // Work split (set by the host per kernel geometry):
  //   body: tiles [0, body_tiles) of every strip, TB bytes each, all via TMA;
  //   tail: bytes [body_tiles*TB, pbytes) via direct loads, chunk_bytes per unit.
  uint64_t body_tiles;
  uint64_t tail_units_per_stripe;
  // != 0: the last body tile of every strip is partial -- this many bytes (a multiple of 16;
  // kernels with FastEntry::partial_tile only, all rows then being `bytes` long)
  uint32_t last_tile;
  // NEXT-1 modes.  update: strip upd[s*upd_stride] (or upd_k) of stripe s is rewritten with
  // the new data at nbase + s*new_stride; scrub: counts[s] += words violating a parity equation.
  const int32_t* upd;
  int upd_rows;  // = 4 (old d_k, new d_k, P, Q); a runtime value on purpose, see num_rows()
  int upd_stride;
  int upd_k;
  const uint8_t* nbase;
  uint64_t new_stride;
  uint32_t* counts;
  // NEXT-2: multiplier programs for the extended code, one per erasure pair
  // (prog[pair_index(x, y, N)]); N > p only.
  const ExtProg* prog;
  // NEXT-4 (cross-GPU stripe layout, include/raid6c.h).  partial: rows = the surviving strips
  // with global index in [k_lo, k_hi); word range g of its two outputs goes to
  // part_p[g] / part_q[g] + s*part_stride + (off - g*range_bytes).
  int k_lo, k_hi;
  int nranges;
  uint64_t range_bytes;
  uint64_t part_stride;
  uint8_t* part_p[RAID6C_MAX_RANKS];
  uint8_t* part_q[RAID6C_MAX_RANKS];
  // combine: bytes [range_lo, range_hi) of every stripe from nsrc partial slots
  // (src_p[r] / src_q[r] + s*part_stride), then the class solve; outputs to base[k].
  int nsrc;
  uint64_t range_lo, range_hi;
  const uint8_t* src_p[RAID6C_MAX_RANKS];
  const uint8_t* src_q[RAID6C_MAX_RANKS];
};

// Kernel-geometry record for one compiled prime (fast path) -- filled by each
// instantiation translation unit and used by the host to split work and launch.
struct FastEntry {
  int p;
  // per kernel mode (the geometry may differ between modes, see zp_fast.cuh Geo):
  int chunk_bytes[7];  // bytes per thread-chunk (whole periods of lcm(n,32) bits)
  int tile_bytes[7];   // TMA row bytes = consumer threads * chunk_bytes
  int threads[7];      // consumer threads (+32 producer threads per CTA)
  // __global__ void(ZpArgs) per mode: encode, recover, scrub, update, partial, combine (NEXT-4),
  // light recovery (classes DP / DQ / PQ only, encode geometry; basic code only)
  const void* kernel[7];
  size_t smem_bytes[7];
  int partial_tile[7];  // the mode's kernel loads / stores a partial last tile through TMA
  const void* kernel_ext[7];  // extended-code (N > p) kernels, nullptr if p fails Theorem 25.3
  size_t smem_ext[7];
};

const FastEntry* fast_entry(int p);  // nullptr if p has no fast path

// Index of the canonical pair (x < y) among the C(N+2, 2) pairs of strip indices, row-major.
__host__ __device__ inline int pair_index(int x, int y, int N) {
  const int K = N + 2;
  return x * (2 * K - x - 1) / 2 + (y - x - 1);
}

// Generic (runtime-p) kernels, any odd prime <= 257.
enum : int { KMODE_ENCODE = 0, KMODE_RECOVER = 1, KMODE_SCRUB = 2, KMODE_UPDATE = 3, KMODE_PARTIAL = 4,
             KMODE_COMBINE = 5, KMODE_RECOVER_L = 6 /* fast path, basic code: launches without DD */ };
constexpr int NUM_KMODES = 7;
cudaError_t generic_launch(const ZpArgs& a, int p, int mode, cudaStream_t st, int num_sms);

}  // namespace zp
