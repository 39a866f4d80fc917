// zp_fast.cuh -- compile-time-p Z_p-RAID kernel for sm_100a (encode and all recovery classes).
//
// What it computes (DESIGN.md section "Path"):
//   encode   P = sum d_i, Q = sum x^i d_i            Eq. (znparity)
//   recover  PQ / DQ / DP / DD classes               Lemma 23.2 proof PAPER.md:380-401,
//                                                    Sec. 4.3/4.6 PAPER.md:965-992, 1124-1160
// over strips that are LSB-first streams of n = p-1 bit words (R1, R2).
//
// How (B200-first; the paper's SSE2 loop is prior art, not the blueprint):
//   * A CTA owns a tile column: the same TB-byte range of all N source strips of one stripe.
//     One producer lane streams the N tile rows HBM -> SMEM with cp.async.bulk (TMA, 1-D),
//     completing on mbarriers; STAGES rows are in flight per CTA.
//   * Each consumer thread owns a chunk of C 32-bit lanes = whole periods of lcm(n,32) bits,
//     so every chunk starts on a word boundary and its word layout is a compile-time
//     constant.  The chunk is processed as a packed bit stream, never unpacked into words:
//       multiplication by x^a (Eq. (powers)) = rotation by a inside each
//       p-bit slot of R' = F2[x]/(x^p+1) followed by the reduction pi (if slot bit p-1 is set,
//       flip bits 0..n-1).  pi is a ring homomorphism R' -> R_p, so it is DEFERRED to once
//       per word per output (not once per disk as in the paper's Horner loop).
//       In stream form, for a = 1..n:   X = S << a (funnel shift across lanes),
//                                        Y = S >> (p - a)
//         ax ^= X & MX(a)   MX(a) = word positions a..n-1, plus position 0 which receives the
//                           slot bit p-1 (the "overflow" T) of the previous word,
//         ay ^= Y & ML(a)   ML(a) = word positions 0..a-2 (the wrapped part).
//       The overflow of the chunk's last word leaves through a virtual lane C (tc).
//     Reduction (once per output): T = overflow bits (at position 0 of word w+1 for word w),
//       F = T - (T >> n) has ones exactly on the words whose T is set; Q = ay ^ (ax & ~M0) ^ F.
//   * Epilogue per class: DQ adds x^j d_j, DP reads its rotated sum directly, DD forms
//     t = dP + x^{-x} dQ and applies (1 + x^z)^{-1} = sum_{m<(p+1)/2} x^{2zm} (PAPER.md:1139-1146,
//     reading R11) by a doubling chain of ~2 log2(p) rotations instead of the paper's
//     (p-1)/2-step Horner series.
//   * Outputs go registers -> SMEM -> cp.async.bulk store (bulk_group).
//   * The ragged end of each strip ([body_tiles*TB, parity_bytes)) is handled by the same
//     arithmetic with direct, byte-precise global loads and stores (tail units).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sub_chain.cuh"
#include "zp_args.h"

namespace zp {

constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
constexpr int top_bit(int v) { return v <= 1 ? 0 : 1 + top_bit(v >> 1); }

template <int P_>
struct Geo {
  static constexpr int P = P_;
  static constexpr int n = P - 1;
  static constexpr int LAMBDA = n / cgcd(n, 32);  // 32-bit lanes per period lcm(n,32)
  static constexpr int C = LAMBDA < 12 ? LAMBDA * (12 / LAMBDA) : LAMBDA;  // lanes per chunk
  static constexpr int CB = 4 * C;                   // chunk bytes
  static constexpr int QMAX = n >> 5;                // max whole-lane shift
  // consumer threads per CTA; 224 for lane-aligned small words (n | 32) so that the 48-byte
  // chunk tiles (10752 B) leave a 1.5% instead of 6% ragged tail on 64 KiB strips (config 1)
  static constexpr int THREADS = C >= 24 ? 128 : ((32 % n == 0) ? 224 : 256);
  static constexpr int TB = THREADS * CB;            // TMA row (tile) bytes
  static constexpr int MTAB = (n + 1) * LAMBDA;      // mask table entries (uint2)
  static constexpr int SMEM_TARGET = 112 * 1024;     // 2 CTAs per SM
  static constexpr int STAGES_RAW = (SMEM_TARGET - 2 * TB - MTAB * 8 - 256) / TB;
  static constexpr int STAGES = STAGES_RAW < 3 ? 3 : (STAGES_RAW > 8 ? 8 : STAGES_RAW);
  static constexpr size_t SMEM = (size_t)(STAGES + 2) * TB + (size_t)MTAB * 8 + 2 * STAGES * 8;
  static_assert(LAMBDA <= 32, "fast path needs a period of at most 32 lanes");
  static_assert(TB % 16 == 0, "TMA rows must be multiples of 16 bytes");
};

// Word-position-0 mask of lane `phi` of a period (compile-time).
template <int n>
__host__ __device__ constexpr uint32_t m0_mask(int phi) {
  uint32_t m = 0;
  for (int b = 0; b < 32; b++)
    if ((32 * phi + b) % n == 0) m |= 1u << b;
  return m;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "ZP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra ZP_WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_row(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ chunk I/O
template <int C>
__device__ __forceinline__ void ld_chunk_smem(const uint8_t* p, uint32_t (&L)[C]) {
  if constexpr ((4 * C) % 16 == 0) {
#pragma unroll
    for (int v = 0; v < C / 4; v++) {
      uint4 t = reinterpret_cast<const uint4*>(p)[v];
      L[4 * v] = t.x; L[4 * v + 1] = t.y; L[4 * v + 2] = t.z; L[4 * v + 3] = t.w;
    }
  } else if constexpr ((4 * C) % 8 == 0) {
#pragma unroll
    for (int v = 0; v < C / 2; v++) {
      uint2 t = reinterpret_cast<const uint2*>(p)[v];
      L[2 * v] = t.x; L[2 * v + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < C; v++) L[v] = reinterpret_cast<const uint32_t*>(p)[v];
  }
}
template <int C>
__device__ __forceinline__ void st_chunk_smem(uint8_t* p, const uint32_t (&L)[C]) {
  if constexpr ((4 * C) % 16 == 0) {
#pragma unroll
    for (int v = 0; v < C / 4; v++)
      reinterpret_cast<uint4*>(p)[v] = make_uint4(L[4 * v], L[4 * v + 1], L[4 * v + 2], L[4 * v + 3]);
  } else if constexpr ((4 * C) % 8 == 0) {
#pragma unroll
    for (int v = 0; v < C / 2; v++) reinterpret_cast<uint2*>(p)[v] = make_uint2(L[2 * v], L[2 * v + 1]);
  } else {
#pragma unroll
    for (int v = 0; v < C; v++) reinterpret_cast<uint32_t*>(p)[v] = L[v];
  }
}
// Direct global chunk load, zero past `len` bytes of the strip (off = chunk offset in strip).
template <int C>
__device__ __forceinline__ void ld_chunk_global(const uint8_t* __restrict__ g, uint64_t off, uint64_t len,
                                                uint32_t (&L)[C]) {
  const bool al4 = (reinterpret_cast<uintptr_t>(g) & 3u) == 0;
#pragma unroll
  for (int l = 0; l < C; l++) {
    const uint64_t o = off + 4u * l;
    if (al4 && o + 4 <= len) {
      L[l] = __ldg(reinterpret_cast<const uint32_t*>(g + 4 * l));
    } else {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; b++)
        if (o + b < len) v |= static_cast<uint32_t>(__ldg(g + 4 * l + b)) << (8 * b);
      L[l] = v;
    }
  }
}
template <int C>
__device__ __forceinline__ void st_chunk_global(uint8_t* __restrict__ g, uint64_t off, uint64_t len,
                                                const uint32_t (&L)[C]) {
  const bool al4 = (reinterpret_cast<uintptr_t>(g) & 3u) == 0;
#pragma unroll
  for (int l = 0; l < C; l++) {
    const uint64_t o = off + 4u * l;
    if (al4 && o + 4 <= len) {
      reinterpret_cast<uint32_t*>(g)[l] = L[l];
    } else {
#pragma unroll
      for (int b = 0; b < 4; b++)
        if (o + b < len) g[4 * l + b] = static_cast<uint8_t>(L[l] >> (8 * b));
    }
  }
}

// ------------------------------------------------------------------ ring arithmetic on a chunk
// Accumulator of a sum of rotated terms in deferred (R') form.
template <class G>
struct Acc {
  uint32_t ax[G::C];
  uint32_t ay[G::C];
  uint32_t tc;
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int l = 0; l < G::C; l++) { ax[l] = 0; ay[l] = 0; }
    tc = 0;
  }
};

// acc += x^a * S for a in [1, n], lane shift Q = a>>5 (left) and QP = (p-a)>>5 (right).
template <class G, int Q, int QP>
__device__ __forceinline__ void rot_body(const uint32_t (&S)[G::C], uint32_t r, uint32_t rp,
                                         const uint2* __restrict__ mrow, Acc<G>& acc) {
  constexpr int C = G::C;
#pragma unroll
  for (int l = 0; l < C; l++) {
    const uint2 m = mrow[l % G::LAMBDA];
    const uint32_t xh = (l - Q >= 0) ? S[l - Q >= 0 ? l - Q : 0] : 0u;
    const uint32_t xl = (l - Q - 1 >= 0) ? S[l - Q - 1 >= 0 ? l - Q - 1 : 0] : 0u;
    const uint32_t X = __funnelshift_l(xl, xh, r);
    acc.ax[l] ^= X & m.x;
    const uint32_t yl = (l + QP < C) ? S[l + QP < C ? l + QP : 0] : 0u;
    const uint32_t yh = (l + QP + 1 < C) ? S[l + QP + 1 < C ? l + QP + 1 : 0] : 0u;
    const uint32_t Y = __funnelshift_r(yl, yh, rp);
    acc.ay[l] ^= Y & m.y;
  }
  // virtual lane C: carries the slot-(p-1) bit of the chunk's last word (bit 0 only matters)
  const uint32_t vh = (C - Q < C) ? S[C - Q < C ? C - Q : 0] : 0u;
  const uint32_t vl = (C - Q - 1 >= 0 && C - Q - 1 < C) ? S[(C - Q - 1 >= 0 && C - Q - 1 < C) ? C - Q - 1 : 0] : 0u;
  acc.tc ^= __funnelshift_l(vl, vh, r);
}

template <class G>
__host__ __device__ constexpr bool reachable(int Q, int QP) {
  for (int a = 1; a <= G::n; a++)
    if ((a >> 5) == Q && ((G::P - a) >> 5) == QP) return true;
  return false;
}

template <class G, int K>
__device__ __forceinline__ void rot_dispatch(int key, const uint32_t (&S)[G::C], uint32_t r, uint32_t rp,
                                             const uint2* __restrict__ mrow, Acc<G>& acc) {
  if constexpr (K < (G::QMAX + 1) * (G::QMAX + 1)) {
    constexpr int Q = K / (G::QMAX + 1);
    constexpr int QP = K % (G::QMAX + 1);
    if constexpr (reachable<G>(Q, QP)) {
      if (key == K) {
        rot_body<G, Q, QP>(S, r, rp, mrow, acc);
        return;
      }
    }
    rot_dispatch<G, K + 1>(key, S, r, rp, mrow, acc);
  }
}

// acc += x^a * S   (a in [0, p), S reduced or not: only its n stream bits are used)
template <class G>
__device__ __forceinline__ void rot_acc(const uint32_t (&S)[G::C], int a, const uint2* __restrict__ mtab, Acc<G>& acc) {
  if (a == 0) {
#pragma unroll
    for (int l = 0; l < G::C; l++) acc.ay[l] ^= S[l];
    return;
  }
  const int q = a >> 5, qp = (G::P - a) >> 5;
  const uint32_t r = static_cast<uint32_t>(a & 31), rp = static_cast<uint32_t>((G::P - a) & 31);
  rot_dispatch<G, 0>(q * (G::QMAX + 1) + qp, S, r, rp, mtab + a * G::LAMBDA, acc);
}

// V = pi(acc): the reduced n-bit stream of the accumulated R' value.
template <class G>
__device__ __forceinline__ void reduce(const Acc<G>& acc, uint32_t (&V)[G::C]) {
  constexpr int C = G::C;
  constexpr int qn = G::n >> 5, rn = G::n & 31;
  uint32_t T[C + 1], Ts[C + 1], F[C + 1];
#pragma unroll
  for (int l = 0; l < C; l++) T[l] = acc.ax[l] & m0_mask<G::n>(l % G::LAMBDA);
  T[C] = acc.tc & 1u;
#pragma unroll
  for (int l = 0; l <= C; l++) {
    const uint32_t lo = (l + qn <= C) ? T[l + qn <= C ? l + qn : 0] : 0u;
    const uint32_t hi = (l + qn + 1 <= C) ? T[l + qn + 1 <= C ? l + qn + 1 : 0] : 0u;
    Ts[l] = rn ? __funnelshift_r(lo, hi, rn) : lo;
  }
  SubChain<C + 1>::run(F, T, Ts);  // F = T - (T >> n): ones on every word whose T is set
#pragma unroll
  for (int l = 0; l < C; l++) V[l] = (acc.ax[l] & ~m0_mask<G::n>(l % G::LAMBDA)) ^ acc.ay[l] ^ F[l];
}

// ------------------------------------------------------------------ stripe bookkeeping
enum : int { CLS_PQ = 0, CLS_DQ = 1, CLS_DP = 2, CLS_DD = 3 };

struct ItemDesc {
  int x, y;   // canonical lost pair, x < y
  int cls;    // CLS_*
  int base;   // rotation origin: amounts are (k - base) mod p
};

template <bool RECOVER>
__device__ __forceinline__ ItemDesc item_desc(const ZpArgs& a, int s) {
  ItemDesc d;
  int i = a.N, j = a.N + 1;
  if constexpr (RECOVER) {
    if (a.er) {
      const int2 e = a.er[static_cast<int64_t>(s) * a.er_stride];
      i = e.x; j = e.y;
    } else {
      i = a.ei; j = a.ej;
    }
  }
  d.x = i < j ? i : j;
  d.y = i < j ? j : i;
  if (d.y == a.N + 1) d.cls = (d.x == a.N) ? CLS_PQ : CLS_DQ;
  else d.cls = (d.y == a.N) ? CLS_DP : CLS_DD;
  d.base = (d.cls == CLS_DP || d.cls == CLS_DD) ? d.x : 0;
  return d;
}

// r-th surviving strip (r in [0, N)), skipping the lost pair.
__device__ __forceinline__ int source_strip(int r, const ItemDesc& d) {
  int k = r;
  if (k >= d.x) k++;
  if (k >= d.y) k++;
  return k;
}

__device__ __forceinline__ uint64_t strip_stride(const ZpArgs& a, int k) {
  return k < a.N ? a.data_stride : a.parity_stride;
}

// Fold one source row into the accumulators (P part and rotated Q part).
template <class G>
__device__ __forceinline__ void fold_row(const ZpArgs& a, const ItemDesc& d, int k, const uint32_t (&L)[G::C],
                                         const uint2* __restrict__ mtab, uint32_t (&Pa)[G::C], Acc<G>& acc) {
  if (k <= a.N) {  // data strips and P feed the P accumulator
#pragma unroll
    for (int l = 0; l < G::C; l++) Pa[l] ^= L[l];
  }
  if (k != a.N) {  // data strips and Q feed the rotated accumulator
    int amt = (k < a.N) ? (k - d.base) : (G::P - d.base);
    amt %= G::P;
    if (amt < 0) amt += G::P;
    rot_acc<G>(L, amt, mtab, acc);
  }
}

// Class epilogue: produces the two output chunks and their strip indices.
template <class G>
__device__ __forceinline__ void finish(const ZpArgs& a, const ItemDesc& d, uint32_t (&Pa)[G::C], Acc<G>& acc,
                                       const uint2* __restrict__ mtab, uint32_t (&o0)[G::C], uint32_t (&o1)[G::C],
                                       int& k0, int& k1) {
  constexpr int C = G::C;
  if (d.cls == CLS_PQ) {  // P, Q re-encoded
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = Pa[l];
    reduce<G>(acc, o1);
    k0 = a.N; k1 = a.N + 1;
  } else if (d.cls == CLS_DQ) {  // d_j = P + sum_{k!=j} d_k; Q += x^j d_j
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = Pa[l];
    rot_acc<G>(o0, d.x, mtab, acc);
    reduce<G>(acc, o1);
    k0 = d.x; k1 = a.N + 1;
  } else if (d.cls == CLS_DP) {  // d_j = x^{-j}(Q + sum_{k!=j} x^k d_k); P = sum
    reduce<G>(acc, o0);
#pragma unroll
    for (int l = 0; l < C; l++) o1[l] = Pa[l] ^ o0[l];
    k0 = d.x; k1 = a.N;
  } else {  // DD: d_y = (1+x^z)^{-1}(dP + x^{-x} dQ), d_x = d_y + dP
#pragma unroll
    for (int l = 0; l < C; l++) acc.ay[l] ^= Pa[l];
    uint32_t t[C];
    reduce<G>(acc, t);
    // S_m = sum_{j<m} b^j t, b = x^{2z}; target m* = (p+1)/2 (reading R11).
    constexpr int M = (G::P + 1) / 2;
    constexpr int TOP = top_bit(M);
    const int bz = (2 * (d.y - d.x)) % G::P;
#pragma unroll
    for (int l = 0; l < C; l++) o1[l] = t[l];  // o1 = S_1
    int m = 1;
#pragma unroll 1
    for (int bit = TOP - 1; bit >= 0; bit--) {
      acc.zero();  // S_{2m} = S_m + b^m S_m
#pragma unroll
      for (int l = 0; l < C; l++) acc.ay[l] = o1[l];
      rot_acc<G>(o1, (bz * m) % G::P, mtab, acc);
      reduce<G>(acc, o1);
      m *= 2;
      if ((M >> bit) & 1) {  // S_{m+1} = S_m + b^m t
        acc.zero();
#pragma unroll
        for (int l = 0; l < C; l++) acc.ay[l] = o1[l];
        rot_acc<G>(t, (bz * m) % G::P, mtab, acc);
        reduce<G>(acc, o1);
        m += 1;
      }
    }
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = o1[l] ^ Pa[l];
    k0 = d.x; k1 = d.y;
  }
}

// ------------------------------------------------------------------ the kernel
template <int P, bool RECOVER>
__global__ void __launch_bounds__(Geo<P>::THREADS + 32, 2) zp_kernel(const __grid_constant__ ZpArgs a) {
  using G = Geo<P>;
  constexpr int C = G::C, CB = G::CB, TB = G::TB, NT = G::THREADS, ST = G::STAGES;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint8_t* outb = smem + (size_t)ST * TB;
  uint2* mtab = reinterpret_cast<uint2*>(outb + 2 * TB);
  uint64_t* full = reinterpret_cast<uint64_t*>(mtab + G::MTAB);
  uint64_t* empty = full + ST;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // Mask table MX(a), ML(a) per lane phase (positions are word-relative, chunk starts at a word).
  for (int e = tid; e < G::MTAB; e += blockDim.x) {
    const int am = e / G::LAMBDA, phi = e % G::LAMBDA;
    uint32_t mx = 0, ml = 0;
    int pos = (32 * phi) % G::n;
    for (int b = 0; b < 32; b++) {
      if (pos >= am || pos == 0) mx |= 1u << b;
      if (pos + 2 <= am) ml |= 1u << b;
      if (++pos == G::n) pos = 0;
    }
    mtab[e] = make_uint2(mx, ml);
  }
  if (tid == 0) {
    for (int s = 0; s < ST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t tiles = a.body_tiles;
  const uint64_t body_items = tiles * static_cast<uint64_t>(a.num_stripes);

  if (warp == NT / 32) {
    // ------------------------------------------------ producer: one lane issues all TMA rows
    if (lane == 0) {
      uint32_t stage = 0, ph = 0;
      for (uint64_t it = blockIdx.x; it < body_items; it += gridDim.x) {
        const int s = static_cast<int>(it / tiles);
        const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
        const ItemDesc d = item_desc<RECOVER>(a, s);
        for (int r = 0; r < a.N; r++) {
          const int k = source_strip(r, d);
          const uint8_t* g = a.base[k] + static_cast<uint64_t>(s) * strip_stride(a, k) + t * TB;
          mbar_wait(&empty[stage], ph ^ 1u);
          mbar_expect_tx(&full[stage], TB);
          tma_load_row(stages + (size_t)stage * TB, g, TB, &full[stage]);
          if (++stage == ST) { stage = 0; ph ^= 1u; }
        }
      }
    }
    return;
  }

  // -------------------------------------------------- consumers: body tiles via the pipeline
  uint32_t stage = 0, ph = 0;
  for (uint64_t it = blockIdx.x; it < body_items; it += gridDim.x) {
    const int s = static_cast<int>(it / tiles);
    const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
    const ItemDesc d = item_desc<RECOVER>(a, s);
    uint32_t Pa[C];
    Acc<G> acc;
    acc.zero();
#pragma unroll
    for (int l = 0; l < C; l++) Pa[l] = 0;
    for (int r = 0; r < a.N; r++) {
      const int k = source_strip(r, d);
      uint32_t L[C];
      mbar_wait(&full[stage], ph);
      ld_chunk_smem<C>(stages + (size_t)stage * TB + tid * CB, L);
      fold_row<G>(a, d, k, L, mtab, Pa, acc);
      // Release the stage only after every loaded lane has been consumed: an mbarrier.arrive
      // issued right after the LDS does not wait for the loads to complete, and the producer's
      // next TMA write (async proxy) can then overwrite the row under a lagging warp's reads.
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == ST) { stage = 0; ph ^= 1u; }
    }
    uint32_t o0[C], o1[C];
    int k0, k1;
    finish<G>(a, d, Pa, acc, mtab, o0, o1, k0, k1);
    if (tid == 0) bulk_wait_read0();  // previous item's bulk stores have read outb
    named_bar_sync(1, NT);
    st_chunk_smem<C>(outb + tid * CB, o0);
    st_chunk_smem<C>(outb + TB + tid * CB, o1);
    fence_proxy_async_smem();
    named_bar_sync(1, NT);
    if (tid == 0) {
      tma_store_row(const_cast<uint8_t*>(a.base[k0]) + static_cast<uint64_t>(s) * strip_stride(a, k0) + t * TB, outb, TB);
      tma_store_row(const_cast<uint8_t*>(a.base[k1]) + static_cast<uint64_t>(s) * strip_stride(a, k1) + t * TB,
                    outb + TB, TB);
      bulk_commit();
    }
  }

  // -------------------------------------------------- tail units: direct byte-precise path
  const uint64_t tups = a.tail_units_per_stripe;
  const uint64_t tail_total = tups * static_cast<uint64_t>(a.num_stripes);
  const uint64_t body_end = tiles * TB;
  for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * NT + tid; u < tail_total;
       u += static_cast<uint64_t>(gridDim.x) * NT) {
    const int s = static_cast<int>(u / tups);
    const uint64_t off = body_end + (u - static_cast<uint64_t>(s) * tups) * CB;
    const ItemDesc d = item_desc<RECOVER>(a, s);
    uint32_t Pa[C];
    Acc<G> acc;
    acc.zero();
#pragma unroll
    for (int l = 0; l < C; l++) Pa[l] = 0;
    for (int r = 0; r < a.N; r++) {
      const int k = source_strip(r, d);
      const uint64_t len = k < a.N ? a.bytes : a.pbytes;
      uint32_t L[C];
      ld_chunk_global<C>(a.base[k] + static_cast<uint64_t>(s) * strip_stride(a, k) + off, off, len, L);
      fold_row<G>(a, d, k, L, mtab, Pa, acc);
    }
    uint32_t o0[C], o1[C];
    int k0, k1;
    finish<G>(a, d, Pa, acc, mtab, o0, o1, k0, k1);
    st_chunk_global<C>(const_cast<uint8_t*>(a.base[k0]) + static_cast<uint64_t>(s) * strip_stride(a, k0) + off, off,
                       k0 < a.N ? a.bytes : a.pbytes, o0);
    st_chunk_global<C>(const_cast<uint8_t*>(a.base[k1]) + static_cast<uint64_t>(s) * strip_stride(a, k1) + off, off,
                       k1 < a.N ? a.bytes : a.pbytes, o1);
  }
  if (tid == 0) bulk_wait0();
}

template <int P>
FastEntry make_entry() {
  using G = Geo<P>;
  FastEntry e;
  e.p = P;
  e.chunk_bytes = G::CB;
  e.tile_bytes = G::TB;
  e.threads = G::THREADS;
  e.smem_bytes = G::SMEM;
  e.enc_kernel = reinterpret_cast<const void*>(&zp_kernel<P, false>);
  e.rec_kernel = reinterpret_cast<const void*>(&zp_kernel<P, true>);
  return e;
}

}  // namespace zp

#define ZP_INSTANTIATE_FAST(PP)                                                   \
  namespace zp {                                                                  \
  template __global__ void zp_kernel<PP, false>(const __grid_constant__ ZpArgs); \
  template __global__ void zp_kernel<PP, true>(const __grid_constant__ ZpArgs);  \
  const FastEntry* fast_entry_##PP() {                                            \
    static const FastEntry e = make_entry<PP>();                                  \
    return &e;                                                                    \
  }                                                                               \
  }
