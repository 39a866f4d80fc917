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
#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

#include "sub_chain.cuh"
#include "tma_ring.cuh"
#include "zp_args.h"

// ZP_BOUNDS_CHECK builds (python -m paper_cs_0611109_b200.build -D ZP_BOUNDS_CHECK --out ...)
// assert that every TMA row load and bulk store stays inside its strip / slot: the stand-in for
// compute-sanitizer, which is closed on this GPU pool.  Off in the product build.
#ifdef ZP_BOUNDS_CHECK
#define ZP_CHECK(cond) assert(cond)
#else
#define ZP_CHECK(cond) ((void)0)
#endif

namespace zp {

constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
constexpr int top_bit(int v) { return v <= 1 ? 0 : 1 + top_bit(v >> 1); }

// Chunk / tile geometry of one kernel instantiation.  SMALL8_ selects, for lane-aligned small
// words (n | 32: p = 3, 5, 17), 32-byte chunks x 256 threads = 8 KiB tiles, which divide
// power-of-two strips exactly (no ragged tail); it is used by the light-ALU modes (encode,
// partial: measured +6% on config 1 and +7% for p = 17) and by the NEXT-4 combine (whose word
// ranges are whole partial tiles), while recovery keeps 48-byte chunks (fewer per-chunk epilogue
// overheads per byte: C8 measured -10% there).
#ifndef ZP_REC_THREADS
#define ZP_REC_THREADS 256
#endif
template <int P_, bool SMALL8_ = false, int MINLANES_ = 12, bool REC_ = false>
struct Geo {
  static constexpr int P = P_;
  static constexpr int n = P - 1;
  static constexpr int LAMBDA = n / cgcd(n, 32);  // 32-bit lanes per period lcm(n,32)
  static constexpr bool SMALL8 = SMALL8_ && (32 % n == 0);
  // lanes per chunk: whole periods, at least 12 lanes (48 B) so that the per-chunk epilogue
  // (reductions, the DD series) is amortised; measured for LAMBDA = 5, 7, 9 (p = 11, 29, 19/37):
  // 15 / 14 / 18 lanes recover at 0.92-1.01 of the copy rate vs 0.73-0.89 with 10 / 7 / 9
  // (words that are whole lanes, n = 32*LAMBDA >= 256 bits: one word per chunk, C = LAMBDA)
  static constexpr bool WIDE = (n % 32 == 0) && LAMBDA >= 8;
  static constexpr int C = SMALL8 ? 8
                         : ((LAMBDA < MINLANES_ && !WIDE) ? LAMBDA * ((MINLANES_ + LAMBDA - 1) / LAMBDA) : LAMBDA);
  static constexpr int CB = 4 * C;                   // chunk bytes
  static constexpr int QMAX = n >> 5;                // max whole-lane shift
  // consumer threads per CTA; 224 for lane-aligned small words (n | 32) with 48-byte chunks so
  // that the tiles (10752 B) leave a 1.5% instead of 6% ragged tail on 64 KiB strips (config 1);
  // 128 for chunks of 20 lanes or more (two CTAs of 160 threads keep 168 registers each: with 256
  // the 96-register cap spills, measured p = 23 / 47 / 89 encode 0.74-0.82 -> 0.97-1.00 and
  // recovery 0.50-0.56 -> 0.76-0.95 of the copy rate; p = 43: encode 1.05 -> 0.98, recovery 0.74 -> 0.78);
  // not below 20 lanes: 128 threads for p = 73, 97, 113, 137, 193, 241 (12-18 lanes) cost recovery 11-31 %
  static constexpr int THREADS = SMALL8 ? 256 : (C >= 20 ? 128 : ((32 % n == 0) ? 224 : (REC_ ? ZP_REC_THREADS : 256)));
  static constexpr int TB = THREADS * CB;            // TMA row (tile) bytes
  // Mask table: MX(a), ML(a) per rotation amount a and lane phase (uint2), or -- when that would
  // take more than 40 KB of shared memory (p = 233: 53 KB, leaving 2 TMA stages at 2 CTAs/SM) --
  // ML(a) alone for a = 0..n+1 (uint32), with MX(a) = ~ML(a+1) | M0 derived in the fold
  // (ML(a+1) = word positions 0..a-1, so its complement plus position 0 is MX(a)).  Not for
  // recovery, whose rotations are the bottleneck: measured p = 233 encode 0.95 -> 1.02 of the
  // copy rate with the half table (3 stages), recovery 0.575 -> 0.553 (one more LOP3 per lane).
  static constexpr bool HALF = (n + 1) * LAMBDA * 8 > 40 * 1024 && !REC_;
  static constexpr int MTAB = HALF ? (n + 2) * LAMBDA : (n + 1) * LAMBDA;  // entries
  static constexpr int MTAB_BYTES = MTAB * (HALF ? 4 : 8);
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

// (MX(a), ML(a)) of lane phase phi from row a of the mask table (see Geo::HALF).
template <class G>
__device__ __forceinline__ uint2 mask_pair(const uint2* __restrict__ mrow, int phi) {
  if constexpr (G::HALF) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(mrow);
    return make_uint2(~r[G::LAMBDA + phi] | m0_mask<G::n>(phi), r[phi]);
  } else {
    return mrow[phi];
  }
}
// Row a of the mask table.
template <class G>
__device__ __forceinline__ const uint2* mask_row(const uint2* __restrict__ mtab, int a) {
  if constexpr (G::HALF) return reinterpret_cast<const uint2*>(reinterpret_cast<const uint32_t*>(mtab) + a * G::LAMBDA);
  else return mtab + a * G::LAMBDA;
}

// acc += x^a * S for a in [1, n], lane shift Q = a>>5 (left) and QP = (p-a)>>5 (right).
template <class G, int Q, int QP>
__device__ __forceinline__ void rot_body(const uint32_t (&S)[G::C], uint32_t r, uint32_t rp,
                                         const uint2* __restrict__ mrow, Acc<G>& acc) {
  constexpr int C = G::C;
#pragma unroll
  for (int l = 0; l < C; l++) {
    const uint2 m = mask_pair<G>(mrow, l % G::LAMBDA);
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

// acc += x^a * S for a in [1, p) (no identity check)
template <class G>
__device__ __forceinline__ void rot_acc_nz(const uint32_t (&S)[G::C], int a, const uint2* __restrict__ mtab,
                                           Acc<G>& acc) {
  if constexpr (G::QMAX == 0 && G::P <= 32) {  // words below 32 bits: no whole-lane shift to dispatch
    rot_body<G, 0, 0>(S, static_cast<uint32_t>(a), static_cast<uint32_t>(G::P - a), mask_row<G>(mtab, a), acc);
  } else {
    const int q = a >> 5, qp = (G::P - a) >> 5;
    const uint32_t r = static_cast<uint32_t>(a & 31), rp = static_cast<uint32_t>((G::P - a) & 31);
    rot_dispatch<G, 0>(q * (G::QMAX + 1) + qp, S, r, rp, mask_row<G>(mtab, a), acc);
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
  rot_acc_nz<G>(S, a, mtab, acc);
}

// V = pi(acc): the reduced n-bit stream of the accumulated R' value.
// (r02, measured: spreading T by a multiply on the FMA pipe for n < 32, or by per-word sign
// spreads for n >= 32, instead of the borrow chain -- no serial dependency -- cost c2 recovery
// 2 % and c5 0.5 %, c4 / c1 unchanged; the chain stays.)
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

// V = pi(acc) + E for a reduced E (the DD syndrome t = dP + x^{-x} dQ): E rides in the last
// three-input XOR of the reduction instead of a separate pass over the accumulator.
template <class G>
__device__ __forceinline__ void reduce_plus(const Acc<G>& acc, const uint32_t (&E)[G::C], uint32_t (&V)[G::C]) {
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
  SubChain<C + 1>::run(F, T, Ts);
#pragma unroll
  for (int l = 0; l < C; l++) V[l] = (acc.ax[l] & ~m0_mask<G::n>(l % G::LAMBDA)) ^ acc.ay[l] ^ (F[l] ^ E[l]);
}

// ------------------------------------------------------------------ stripe bookkeeping
enum : int { CLS_PQ = 0, CLS_DQ = 1, CLS_DP = 2, CLS_DD = 3, CLS_SCRUB = 4, CLS_UPDATE = 5 };
// Kernel modes (compile-time): the method's two operations and the NEXT-1 pair around them.
// MODE_PARTIAL (NEXT-4): the fold of a recovery (or encode) restricted to the strips held by one
// rank, stored unsolved as partial syndromes (dP_r, dQ_r) into the word-range owners' slots.
// MODE_COMBINE (NEXT-4): the owner of a word range folds the 2*nsrc partial rows of its slots
// (row 2r = dP_r, row 2r+1 = dQ_r, already reduced) and runs the recovery epilogue.
// MODE_RECOVER_L: recovery of launches without a DD stripe (classes DP, DQ, PQ: the epilogue is
// one reduction and at most one rotation), built with the encode geometry and CTAs per SM
enum : int { MODE_ENCODE = 0, MODE_RECOVER = 1, MODE_SCRUB = 2, MODE_UPDATE = 3, MODE_PARTIAL = 4, MODE_COMBINE = 5,
             MODE_RECOVER_L = 6 };
constexpr int NUM_MODES = 7;
// Geometry of mode MODE's kernel for prime P (see Geo).
// Recovery chunks of at least 15 lanes for p = 7, 13, 17 (measured r01: c2 recovery 0.96 -> 1.01
// of the copy rate, p = 17 0.93 -> 0.98, p = 7 1.02 -> 1.05); not for p = 5 (config 1's 64 KiB
// strips would get a 13 KiB tile with a long ragged tail: 0.91 -> 0.66) nor p = 29 (21 lanes
// spill: 1.02 -> 0.83).
template <int P>
__host__ __device__ constexpr int recover_min_lanes() {
  return (P == 7 || P == 13 || P == 17) ? 15 : 12;
}
template <int P, int MODE>
using GeoM = Geo<P, MODE == MODE_ENCODE || MODE == MODE_RECOVER_L || MODE == MODE_PARTIAL || MODE == MODE_COMBINE,
                 MODE == MODE_RECOVER ? recover_min_lanes<P>() : 12, MODE == MODE_RECOVER>;
constexpr int K_NEW = -1;     // row index of the update's new-data buffer
constexpr int K_PART_P = -2;  // partial-mode outputs (slots of the word-range owners)
constexpr int K_PART_Q = -3;

struct ItemDesc {
  int x, y;   // canonical lost pair, x < y (update: x = the rewritten strip)
  int cls;    // CLS_*
  int base;   // rotation origin: amounts are (k - base) mod p
};

template <int MODE, bool EXT = false>
__device__ __forceinline__ ItemDesc item_desc(const ZpArgs& a, int s) {
  ItemDesc d;
  if constexpr (MODE == MODE_SCRUB) {
    d.x = d.y = -1;
    d.cls = CLS_SCRUB;
    d.base = 0;
    return d;
  } else if constexpr (MODE == MODE_UPDATE) {
    d.x = a.upd ? a.upd[static_cast<int64_t>(s) * a.upd_stride] : a.upd_k;
    d.y = -1;
    d.cls = CLS_UPDATE;
    d.base = 0;
    return d;
  } else {
    int i = a.N, j = a.N + 1;
    if constexpr (MODE == MODE_RECOVER || MODE == MODE_RECOVER_L || MODE == MODE_PARTIAL || MODE == MODE_COMBINE) {
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
    // basic code: move the rotation origin to the lost strip (x^{-x} folded into the amounts);
    // extended code: origin 0, the solve multiplies by a host-computed u (ExtProg)
    d.base = (!EXT && (d.cls == CLS_DP || d.cls == CLS_DD)) ? d.x : 0;
    return d;
  }
}

template <int MODE>
__device__ __forceinline__ int num_rows(const ZpArgs& a, const ItemDesc& d) {
  if constexpr (MODE == MODE_SCRUB) return a.N + 2;     // every strip of the stripe
  // the surviving strips held by this rank: global indices [k_lo, k_hi) minus the lost pair
  else if constexpr (MODE == MODE_PARTIAL)
    return a.k_hi - a.k_lo - (d.x >= a.k_lo && d.x < a.k_hi) - (d.y >= a.k_lo && d.y < a.k_hi);
  else if constexpr (MODE == MODE_COMBINE) return 2 * a.nsrc;  // (dP_r, dQ_r) per source rank
  // old d_k, new d_k, P, Q: the count (4) comes from the launch args so that the compiler keeps
  // the row loop rolled (a compile-time 4 unrolls it and spills the accumulators)
  else if constexpr (MODE == MODE_UPDATE) return a.upd_rows;
  else return a.N;                                      // the N surviving strips
}

// r-th surviving strip (r in [0, N)), skipping the lost pair.
__device__ __forceinline__ int source_strip(int r, const ItemDesc& d) {
  int k = r;
  if (k >= d.x) k++;
  if (k >= d.y) k++;
  return k;
}

// Strip index read by row r (K_NEW = the update's new-data buffer).
// r-th surviving strip at or above k_lo (partial mode), skipping the lost pair (x < y).
__device__ __forceinline__ int source_strip_from(int r, int k_lo, const ItemDesc& d) {
  int k = k_lo + r;
  if (d.x >= k_lo && k >= d.x) k++;
  if (d.y >= k_lo && k >= d.y) k++;
  return k;
}

template <int MODE>
__device__ __forceinline__ int row_strip(const ZpArgs& a, int r, const ItemDesc& d) {
  if constexpr (MODE == MODE_SCRUB) return r;
  else if constexpr (MODE == MODE_PARTIAL) return source_strip_from(r, a.k_lo, d);
  else if constexpr (MODE == MODE_UPDATE) return r == 0 ? d.x : (r == 1 ? K_NEW : a.N + r - 2);
  else return source_strip(r, d);
}

__device__ __forceinline__ uint64_t strip_stride(const ZpArgs& a, int k) {
  return k < a.N ? a.data_stride : a.parity_stride;
}
__device__ __forceinline__ const uint8_t* row_ptr(const ZpArgs& a, int k, int s) {
  return k == K_NEW ? a.nbase + static_cast<uint64_t>(s) * a.new_stride
                    : a.base[k] + static_cast<uint64_t>(s) * strip_stride(a, k);
}
// Length of row k: data strips and the update's new-data row are `bytes` long; P, Q and the
// NEXT-4 partial slots hold parity-format strips (pbytes).
__device__ __forceinline__ uint64_t row_len(const ZpArgs& a, int k) {
  return (k == K_NEW || (k >= 0 && k < a.N)) ? a.bytes : a.pbytes;
}
// Address of tile/chunk offset `off` of source row r (combine: offset inside the word range of
// the partial slot of source r/2; other modes: offset inside strip row_strip(r)).
template <int MODE>
__device__ __forceinline__ const uint8_t* in_ptr(const ZpArgs& a, int r, const ItemDesc& d, int s, uint64_t off) {
  if constexpr (MODE == MODE_COMBINE) {
    const uint8_t* base = (r & 1) ? a.src_q[r >> 1] : a.src_p[r >> 1];
    return base + static_cast<uint64_t>(s) * a.part_stride + off;
  } else {
    return row_ptr(a, row_strip<MODE>(a, r, d), s) + off;
  }
}

// Output address of byte `off` of output strip k of stripe s (partial outputs: the slot of the
// owner of the word range containing `off`; ranges are whole tiles, so a tile has one owner).
__device__ __forceinline__ uint8_t* out_ptr(const ZpArgs& a, int k, int s, uint64_t off) {
  if (k == K_PART_P || k == K_PART_Q) {
    const int g = static_cast<int>(off / a.range_bytes);
    uint8_t* base = (k == K_PART_P) ? a.part_p[g] : a.part_q[g];
    return base + static_cast<uint64_t>(s) * a.part_stride + (off - static_cast<uint64_t>(g) * a.range_bytes);
  }
  return const_cast<uint8_t*>(row_ptr(a, k, s)) + off;
}

// acc += g_k * S for the extended code's coefficient of data strip k (Eq. (qext)):
// x^k for k < p, 1 + x^{k-p+1} for k >= p.
template <class G>
__device__ __forceinline__ void add_ext_coeff(const uint32_t (&S)[G::C], int k, const uint2* __restrict__ mtab,
                                              Acc<G>& acc) {
  if (k < G::P) {
    rot_acc<G>(S, k, mtab, acc);
  } else {
    rot_acc<G>(S, 0, mtab, acc);
    rot_acc<G>(S, k - G::P + 1, mtab, acc);
  }
}

// Fold one source row into the accumulators (P part and rotated Q part).
template <class G, bool EXT = false>
__device__ __forceinline__ void fold_row(const ZpArgs& a, const ItemDesc& d, int k, const uint32_t (&L)[G::C],
                                         const uint2* __restrict__ mtab, uint32_t (&Pa)[G::C], Acc<G>& acc) {
  if (k <= a.N) {  // data strips and P feed the P accumulator
#pragma unroll
    for (int l = 0; l < G::C; l++) Pa[l] ^= L[l];
  }
  if (k != a.N) {  // data strips and Q feed the rotated accumulator
    if constexpr (EXT) {
      if (k < a.N) add_ext_coeff<G>(L, k, mtab, acc);
      else rot_acc<G>(L, 0, mtab, acc);  // Q
    } else {
      int amt = (k < a.N) ? (k - d.base) : (G::P - d.base);
      amt %= G::P;
      if (amt < 0) amt += G::P;
      rot_acc<G>(L, amt, mtab, acc);
    }
  }
}

// The consumer side of one body item of encode / recovery (basic code), row by row in the
// producer's order: the data strips k < N without the lost pair, then P, then Q (each if it
// survives).  Data rows feed P and Q, P feeds P, Q feeds Q; the rotation amount
// (k - base) mod p is carried from strip to strip (Q's is (p - base) mod p = the amount of
// k = 0), so the per-row work is the wait, the chunk load, the fold and the release only.
template <class G, int ST>
__device__ __forceinline__ void fold_item(const ZpArgs& a, const ItemDesc& d, const uint8_t* my_stages,
                                          uint32_t full_sa, uint32_t empty_sa, const uint2* __restrict__ mtab,
                                          int lane, uint32_t& stage, uint32_t& ph, uint32_t (&Pa)[G::C],
                                          Acc<G>& acc) {
  constexpr int C = G::C;
  auto next_row = [&](uint32_t (&L)[C]) {
    mbar_wait_sa(full_sa + 8u * stage, ph);
    ld_chunk_smem<C>(my_stages + static_cast<size_t>(stage) * G::TB, L);
  };
  auto release = [&]() {
    consumer_release(empty_sa + 8u * stage, lane);
    if (++stage == ST) { stage = 0; ph ^= 1u; }
  };
  const int amt0 = d.base == 0 ? 0 : G::P - d.base;  // (0 - base) mod p
  int amt = amt0, k = 0;
  if (amt0 == 0) {  // base 0 (encode, PQ, DQ): strip 0 (if it survives) enters Q as x^0 d_0
    if (d.x != 0) {
      uint32_t L[C];
      next_row(L);
#pragma unroll
      for (int l = 0; l < C; l++) { Pa[l] ^= L[l]; acc.ay[l] ^= L[l]; }
      release();
    }
    k = amt = 1;
  }
  // from here amt != 0 on every surviving strip: it is 0 only at k = base, a lost strip
  for (; k < a.N; k++) {
    if (k != d.x && k != d.y) {
      uint32_t L[C];
      next_row(L);
#pragma unroll
      for (int l = 0; l < C; l++) Pa[l] ^= L[l];
      rot_acc_nz<G>(L, amt, mtab, acc);
      release();
    }
    amt = amt + 1 == G::P ? 0 : amt + 1;
  }
  if (d.x != a.N && d.y != a.N) {  // P
    uint32_t L[C];
    next_row(L);
#pragma unroll
    for (int l = 0; l < C; l++) Pa[l] ^= L[l];
    release();
  }
  if (d.y != a.N + 1) {  // Q
    uint32_t L[C];
    next_row(L);
    rot_acc<G>(L, amt0, mtab, acc);
    release();
  }
}

// The same walk for the extended code (Eq. (qext), NEXT-2): rotation origin 0, data strip k
// enters Q as x^k (k < p) or (1 + x^{k-p+1}) (k >= p; k-p+1 in [1, p-1]), Q as itself.
template <class G, int ST>
__device__ __forceinline__ void fold_item_ext(const ZpArgs& a, const ItemDesc& d, const uint8_t* my_stages,
                                              uint32_t full_sa, uint32_t empty_sa, const uint2* __restrict__ mtab,
                                              int lane, uint32_t& stage, uint32_t& ph, uint32_t (&Pa)[G::C],
                                              Acc<G>& acc) {
  constexpr int C = G::C;
  auto next_row = [&](uint32_t (&L)[C]) {
    mbar_wait_sa(full_sa + 8u * stage, ph);
    ld_chunk_smem<C>(my_stages + static_cast<size_t>(stage) * G::TB, L);
  };
  auto release = [&]() {
    consumer_release(empty_sa + 8u * stage, lane);
    if (++stage == ST) { stage = 0; ph ^= 1u; }
  };
  for (int k = 0; k < a.N; k++) {
    if (k == d.x || k == d.y) continue;
    uint32_t L[C];
    next_row(L);
    if (k == 0 || k >= G::P) {
#pragma unroll
      for (int l = 0; l < C; l++) { Pa[l] ^= L[l]; acc.ay[l] ^= L[l]; }
    } else {
#pragma unroll
      for (int l = 0; l < C; l++) Pa[l] ^= L[l];
    }
    if (k != 0) rot_acc_nz<G>(L, k < G::P ? k : k - G::P + 1, mtab, acc);
    release();
  }
  if (d.x != a.N && d.y != a.N) {  // P
    uint32_t L[C];
    next_row(L);
#pragma unroll
    for (int l = 0; l < C; l++) Pa[l] ^= L[l];
    release();
  }
  if (d.y != a.N + 1) {  // Q
    uint32_t L[C];
    next_row(L);
#pragma unroll
    for (int l = 0; l < C; l++) acc.ay[l] ^= L[l];
    release();
  }
}

// Combine fold: row 2r is source r's dP part, row 2r+1 its dQ part (reduced words: rotation 0).
template <class G>
__device__ __forceinline__ void fold_partial(int r, const uint32_t (&L)[G::C], uint32_t (&Pa)[G::C], Acc<G>& acc) {
  if (r & 1) {
#pragma unroll
    for (int l = 0; l < G::C; l++) acc.ay[l] ^= L[l];
  } else {
#pragma unroll
    for (int l = 0; l < G::C; l++) Pa[l] ^= L[l];
  }
}

// out = u * t for a host-computed ring element u = sum_i x^{e_i} (ExtProg), t reduced.
template <class G>
__device__ __forceinline__ void mul_prog(const uint32_t (&t)[G::C], const ExtProg* __restrict__ pr,
                                         const uint2* __restrict__ mtab, uint32_t (&out)[G::C]) {
  Acc<G> acc;
  acc.zero();
  const int nu = pr->nu;
#pragma unroll 1
  for (int i = 0; i < nu; i++) rot_acc<G>(t, pr->e[i], mtab, acc);
  reduce<G>(acc, out);
}

// Evaluation plan for the geometric series S_M = sum_{m<M} b^m of the DD solve, by a per-lane
// cost model (rotation ~4 ops, reduction ~6 ops): the doubling chain costs a rotation and a
// reduction per step; a two-level split M = M1*M2 + R costs (M2-1) + (M1-1) + R rotations and
// two reductions (M-1 and one if M2 == M).  p = 3, 5, 7: direct; 13: 3x2+1 (c2 recovery +0.3%
// over direct); 17: 3x3; 59: 5x6; 61, 257: chain (8 steps).
constexpr int c_popcount(int v) { return v == 0 ? 0 : (v & 1) + c_popcount(v >> 1); }
template <int M>
struct SeriesPlan {
  // rotations by x^0 (the first term of each level) are free XORs: only the others count
  static constexpr int cost2(int m2) {
    return m2 >= M ? 4 * (M - 1) + 6 : 4 * ((m2 - 1) + (M / m2 - 1) + M % m2) + 12;
  }
  static constexpr int best_m2() {
    int best = M, bc = cost2(M);
    for (int m2 = 2; m2 < M; m2++)
      if (cost2(m2) < bc) { bc = cost2(m2); best = m2; }
    return best;
  }
  static constexpr int M2 = best_m2();
  static constexpr int M1 = M / M2;
  static constexpr int CHAIN_COST = 10 * (top_bit(M) + c_popcount(M) - 1);
  // p = 61 (M = 31) keeps the chain: measured (r01 A/B), the two-level plan spills at the
  // 96-register cap of its 15-lane chunks and ran 1% slower on config 5; elsewhere it wins
  // (c2 recover +1.5%, c4 DD +1.6%, p = 17 recover +3.2%).  Long series (M > 50, p >= 101) take
  // the chain: the model underrates the two-level plan's register cost there (measured recovery,
  // chain vs two-level: p = 101 +5 %, 113 +8 %, 241 +10 %, 109 -1 %; 137, 193 already chain, +17-19 %).
  static constexpr bool CHAIN = (M == 31) || M > 50 || CHAIN_COST < cost2(M2);
};


// out = sum_{m<M} x^{bz*m + e0} t, M = (p+1)/2: the DD solve (1 + x^z)^{-1} = sum_{m<M} x^{2zm}
// (reading R11) with b = x^{bz}, bz = 2z, times x^{e0}.  The evaluation
// order is chosen at compile time (SeriesPlan): direct, two-level, or doubling chain; e0 is
// folded into the rotation amounts of the first level (the chain pays one rotation for it).
// Basic-code form (e0 = 0): every rotation amount bz*j mod p is nonzero (p prime, bz != 0), and
// each level's x^0 term is peeled out of the runtime loop, so it initialises the accumulator
// (no zeroing pass, no identity-rotation branch).
template <class G>
__device__ __forceinline__ void series_apply0(const uint32_t (&t)[G::C], int bz, const uint2* __restrict__ mtab,
                                              Acc<G>& acc, uint32_t (&out)[G::C]) {
  constexpr int C = G::C;
  constexpr int M = (G::P + 1) / 2;
  constexpr int TOP = top_bit(M);
  using SP = SeriesPlan<M>;
  auto start = [&](const uint32_t (&B)[C]) {  // acc = B (the x^0 term)
#pragma unroll
    for (int l = 0; l < C; l++) { acc.ax[l] = 0u; acc.ay[l] = B[l]; }
    acc.tc = 0u;
  };
  if constexpr (!SP::CHAIN) {
    // two-level: S = sum_{i<M1} b^{i M2} T + sum_{m=M1 M2}^{M-1} b^m t, T = sum_{j<M2} b^j t
    uint32_t T[C];
    start(t);
#pragma unroll 1
    for (int j = 1; j < SP::M2; j++) rot_acc_nz<G>(t, (bz * j) % G::P, mtab, acc);
    if constexpr (SP::M2 == M) {
      reduce<G>(acc, out);
    } else {
      reduce<G>(acc, T);
      start(T);
#pragma unroll 1
      for (int i = 1; i < SP::M1; i++) rot_acc_nz<G>(T, (bz * SP::M2 * i) % G::P, mtab, acc);
#pragma unroll 1
      for (int m = SP::M1 * SP::M2; m < M; m++) rot_acc_nz<G>(t, (bz * m) % G::P, mtab, acc);
      reduce<G>(acc, out);
    }
  } else {
#pragma unroll
    for (int l = 0; l < C; l++) out[l] = t[l];  // S_1 = t
    int m = 1;
#pragma unroll 1
    for (int bit = TOP - 1; bit >= 0; bit--) {
      start(out);  // S_{2m} = S_m + b^m S_m
      rot_acc_nz<G>(out, (bz * m) % G::P, mtab, acc);
      reduce<G>(acc, out);
      m *= 2;
      if ((M >> bit) & 1) {  // S_{m+1} = S_m + b^m t
        start(out);
        rot_acc_nz<G>(t, (bz * m) % G::P, mtab, acc);
        reduce<G>(acc, out);
        m += 1;
      }
    }
  }
}

template <class G>
__device__ __forceinline__ void series_apply(const uint32_t (&t)[G::C], int bz, int e0,
                                             const uint2* __restrict__ mtab, Acc<G>& acc, uint32_t (&out)[G::C]) {
  constexpr int C = G::C;
  constexpr int M = (G::P + 1) / 2;
  constexpr int TOP = top_bit(M);
  using SP = SeriesPlan<M>;
  if constexpr (!SP::CHAIN) {
    // two-level: S = sum_{i<M1} b^{i M2} T + sum_{m=M1 M2}^{M-1} b^m x^{e0} t,
    // T = sum_{j<M2} b^j x^{e0} t (direct when M2 == M); one deferred accumulator per level
    uint32_t T[C];
    acc.zero();
#pragma unroll 1
    for (int j = 0; j < SP::M2; j++) rot_acc<G>(t, (bz * j + e0) % G::P, mtab, acc);
    if constexpr (SP::M2 == M) {
      reduce<G>(acc, out);
    } else {
      reduce<G>(acc, T);
      acc.zero();
#pragma unroll 1
      for (int i = 0; i < SP::M1; i++) rot_acc<G>(T, (bz * SP::M2 * i) % G::P, mtab, acc);
#pragma unroll 1
      for (int m = SP::M1 * SP::M2; m < M; m++) rot_acc<G>(t, (bz * m + e0) % G::P, mtab, acc);
      reduce<G>(acc, out);
    }
    return;
  }
  if (e0 == 0) {
#pragma unroll
    for (int l = 0; l < C; l++) out[l] = t[l];  // S_1 = t
  } else {
    acc.zero();
    rot_acc<G>(t, e0, mtab, acc);
    reduce<G>(acc, out);  // S_1 = x^{e0} t
  }
  int m = 1;
#pragma unroll 1
  for (int bit = TOP - 1; bit >= 0; bit--) {
    acc.zero();  // S_{2m} = S_m + b^m S_m
#pragma unroll
    for (int l = 0; l < C; l++) acc.ay[l] = out[l];
    rot_acc<G>(out, (bz * m) % G::P, mtab, acc);
    reduce<G>(acc, out);
    m *= 2;
    if ((M >> bit) & 1) {  // S_{m+1} = S_m + b^m x^{e0} t
      acc.zero();
#pragma unroll
      for (int l = 0; l < C; l++) acc.ay[l] = out[l];
      rot_acc<G>(t, (bz * m + e0) % G::P, mtab, acc);
      reduce<G>(acc, out);
      m += 1;
    }
  }
}

// Extended-code class epilogue (Lemma 23.2 proof, with g_k of Eq. (qext)):
//   PQ: re-encode;  DQ: d_j = P + sum d_k, Q += g_j d_j;
//   DP: d_j = u (Q + sum_{k!=j} g_k d_k), u = g_j^{-1};  P = sum d_k
//   DD: d_y = u (g_x dP + dQ), u = (g_x + g_y)^{-1};  d_x = d_y + dP
template <class G>
__device__ __forceinline__ void finish_ext(const ZpArgs& a, const ItemDesc& d, int s, uint32_t (&Pa)[G::C], Acc<G>& acc,
                                           const uint2* __restrict__ mtab, uint32_t (&o0)[G::C],
                                           uint32_t (&o1)[G::C], int& k0, int& k1) {
  constexpr int C = G::C;
  const ExtProg* pr = a.prog + pair_index(d.x, d.y, a.N);
  if (d.cls == CLS_PQ) {
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = Pa[l];
    reduce<G>(acc, o1);
    k0 = a.N; k1 = a.N + 1;
  } else if (d.cls == CLS_DQ) {
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = Pa[l];
    add_ext_coeff<G>(o0, d.x, mtab, acc);
    reduce<G>(acc, o1);
    k0 = d.x; k1 = a.N + 1;
  } else if (d.cls == CLS_DP) {
    uint32_t t[C];
    reduce<G>(acc, t);
    if (pr->geo_bz) series_apply<G>(t, pr->geo_bz, pr->geo_e0, mtab, acc, o0);  // u = (1 + x^c)^{-1}
    else mul_prog<G>(t, pr, mtab, o0);
#pragma unroll
    for (int l = 0; l < C; l++) o1[l] = Pa[l] ^ o0[l];
    k0 = d.x; k1 = a.N;
  } else {
    add_ext_coeff<G>(Pa, d.x, mtab, acc);
    uint32_t t[C];
    reduce<G>(acc, t);
    // g_x + g_y = x^e (1 + x^z) when both coefficients are monomials or both are binomials
    // 1 + x^c: the basic code's geometric series (host sets geo_bz = 2z, geo_e0 = -e mod p);
    // mixed pairs x^a + 1 + x^c use the host-computed inverse (ExtProg exponents)
    if (pr->geo_bz) series_apply<G>(t, pr->geo_bz, pr->geo_e0, mtab, acc, o1);
    else mul_prog<G>(t, pr, mtab, o1);
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = o1[l] ^ Pa[l];
    k0 = d.x; k1 = d.y;
  }
}

// Number of words of a chunk with a nonzero bit in V (compile-time word layout).
template <class G>
__device__ __forceinline__ uint32_t count_nonzero_words(const uint32_t (&V)[G::C]) {
  constexpr int WORDS = 32 * G::C / G::n;
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < WORDS; w++) {
    const int b0 = w * G::n, b1 = b0 + G::n;
    uint32_t any = 0;
#pragma unroll
    for (int l = b0 / 32; l <= (b1 - 1) / 32; l++) {
      const int lo = b0 > 32 * l ? b0 - 32 * l : 0;
      const int hi = b1 < 32 * l + 32 ? b1 - 32 * l : 32;
      const uint32_t m = (hi - lo == 32) ? 0xFFFFFFFFu : (((1u << (hi - lo)) - 1u) << lo);
      any |= V[l] & m;
    }
    cnt += any != 0u;
  }
  return cnt;
}

// Class epilogue: produces the two output chunks and their strip indices.
template <class G, bool DD = true>
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
  } else if (!DD || d.cls == CLS_DP) {  // d_j = x^{-j}(Q + sum_{k!=j} x^k d_k); P = sum
    reduce<G>(acc, o0);
#pragma unroll
    for (int l = 0; l < C; l++) o1[l] = Pa[l] ^ o0[l];
    k0 = d.x; k1 = a.N;
  } else if constexpr (DD) {  // DD: d_y = (1+x^z)^{-1}(dP + x^{-x} dQ), d_x = d_y + dP
    uint32_t t[C];
    reduce_plus<G>(acc, Pa, t);
    // d_y = S_M t with S_M = sum_{m<M} b^m, b = x^{2z}, M = (p+1)/2 (reading R11)
    series_apply0<G>(t, (2 * (d.y - d.x)) % G::P, mtab, acc, o1);
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = o1[l] ^ Pa[l];
    k0 = d.x; k1 = d.y;
  }
}

// ------------------------------------------------------------------ the kernel
template <int MODE>
__host__ __device__ constexpr int num_outputs() {
  return MODE == MODE_SCRUB ? 0 : (MODE == MODE_UPDATE ? 3 : 2);
}

// Mask table MX(a), ML(a) per lane phase (positions are word-relative, chunk starts at a word).
template <class G>
__device__ __forceinline__ void build_mtab(uint2* mtab) {
  for (int e = threadIdx.x; e < G::MTAB; e += blockDim.x) {
    const int am = e / G::LAMBDA, phi = e % G::LAMBDA;
    uint32_t mx = 0, ml = 0;
    int pos = (32 * phi) % G::n;
    for (int b = 0; b < 32; b++) {
      if (pos >= am || pos == 0) mx |= 1u << b;
      if (pos + 2 <= am) ml |= 1u << b;
      if (++pos == G::n) pos = 0;
    }
    if constexpr (G::HALF) reinterpret_cast<uint32_t*>(mtab)[e] = ml;
    else mtab[e] = make_uint2(mx, ml);
  }
}

// Shared-memory layout per (p, mode): STAGES TMA rows, NOUT output rows, mask table, barriers.
// CTAs per SM that the kernel of (P, MODE) is built for: the register cap of
// __launch_bounds__ and the shared-memory budget per CTA (112 KB for 2, 72 KB for 3).  Measured
// (r01 A/B): encode of 6-, 12- and 256-bit words gains from a third CTA (p = 13: 0.97 -> 1.06 of
// the copy rate, p = 7: 0.98 -> 1.08, p = 257: 1.02 -> 1.05; 72 registers), and the NEXT-4
// partial (+0-4%) and NEXT-1 update (c2 +2%, c3 +11%) with it, while every recovery mode, the
// scrub (c3 -5%) and the other primes' encode lose with it
// (spills at 128 / 72 registers for p = 59 / 61, a 63-register cap for the 8 KiB-tile primes).
template <int P, int MODE>
__host__ __device__ constexpr int min_blocks() {
  return ((P == 7 || P == 13 || P == 257) &&
          (MODE == MODE_ENCODE || MODE == MODE_RECOVER_L || MODE == MODE_PARTIAL || MODE == MODE_UPDATE))
             ? 3 : 2;
}

template <int P, int MODE>
struct Layout {
  using G = GeoM<P, MODE>;
  static constexpr int NOUT = num_outputs<MODE>();
  static constexpr int SMEM_TARGET = min_blocks<P, MODE>() == 3 ? 72 * 1024 : 112 * 1024;
  static constexpr int STAGES_RAW = (SMEM_TARGET - NOUT * G::TB - G::MTAB_BYTES - 256) / G::TB;
  static constexpr size_t smem_for(int st) {
    return (size_t)(st + NOUT) * G::TB + (size_t)G::MTAB_BYTES + 2 * st * 8;
  }
  static constexpr bool fits(int st) { return (smem_for(st) + 1024) * min_blocks<P, MODE>() <= 228 * 1024; }
  // at least 3 stages; 2 only where 3 would cost a CTA per SM (large mask tables: p = 233
  // encode / recovery, the update of p = 73, 137, 241)
  static constexpr int STAGES = STAGES_RAW >= 3 ? (STAGES_RAW > 8 ? 8 : STAGES_RAW) : (!fits(3) && fits(2) ? 2 : 3);
  static constexpr size_t SMEM = smem_for(STAGES);
  // CTAs per SM that the shared memory actually admits (228 KB per SM, 1 KB reserved per CTA);
  // the launch bounds take this, not the wish of min_blocks (p = 233 update: 1).
  static constexpr int SMEM_FIT = static_cast<int>((228 * 1024) / (SMEM + 1024));
  static constexpr int BLOCKS = SMEM_FIT < min_blocks<P, MODE>() ? SMEM_FIT : min_blocks<P, MODE>();
  static_assert(SMEM <= 227 * 1024 && BLOCKS >= 1, "one CTA must fit the SM's shared memory");
};

// Kernels that finish a short strip end with a partial TMA tile (ZpArgs::last_tile): encode and
// recovery of lane-aligned words (n | 32: p = 3, 5, 17 -- config 1's 64 KiB strips leave 1 KiB
// after the last whole tile).  Other kernels keep the direct tail path: r01 measured the partial
// tile in every kernel at -3..6 % elsewhere (code size), so it is compiled in only here.
template <int P, int MODE, bool EXT>
__host__ __device__ constexpr bool has_partial_tile() {
#ifdef ZP_NO_PARTIAL_TILE  // A/B control
  return false;
#else
  return (32 % (P - 1) == 0) && (MODE == MODE_ENCODE || MODE == MODE_RECOVER || MODE == MODE_RECOVER_L) && !EXT;
#endif
}

// Per-item epilogue for every mode: fills the NOUT output chunks and their strip indices
// (scrub: adds the count of words violating a parity equation to a.counts[s]).
template <int MODE, class G, bool WARP_UNIFORM = true, bool EXT = false>
__device__ __forceinline__ void epilogue(const ZpArgs& a, const ItemDesc& d, int s, uint32_t (&Pa)[G::C], Acc<G>& acc,
                                         const uint32_t (&NEW)[G::C], const uint2* __restrict__ mtab,
                                         uint32_t (&o0)[G::C], uint32_t (&o1)[G::C], int& k0, int& k1, int& k2) {
  constexpr int C = G::C;
  if constexpr (MODE == MODE_SCRUB) {
    // syndromes of both parity equations (Eq. (znparity)): S_P = P + sum d_i, S_Q = Q + sum x^i d_i
    reduce<G>(acc, o1);
#pragma unroll
    for (int l = 0; l < C; l++) o1[l] |= Pa[l];
    uint32_t bad = count_nonzero_words<G>(o1);
    if constexpr (WARP_UNIFORM) {  // body items: the whole warp works on stripe s
      bad = __reduce_add_sync(0xffffffffu, bad);
      if ((threadIdx.x & 31) == 0 && bad) atomicAdd(a.counts + s, bad);
    } else if (bad) {
      atomicAdd(a.counts + s, bad);
    }
  } else if constexpr (MODE == MODE_UPDATE) {
    // P' = P + (old + new), Q' = Q + x^k (old + new)  (linearity of Eq. (znparity)); d_k' = new
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = Pa[l];
    reduce<G>(acc, o1);
    k0 = a.N; k1 = a.N + 1; k2 = d.x;
  } else if constexpr (MODE == MODE_PARTIAL) {
    // unsolved partial syndromes; pi is a homomorphism, so reduced partials add up (NEXT-4)
#pragma unroll
    for (int l = 0; l < C; l++) o0[l] = Pa[l];
    reduce<G>(acc, o1);
    k0 = K_PART_P; k1 = K_PART_Q;
  } else if constexpr (EXT) {
    finish_ext<G>(a, d, s, Pa, acc, mtab, o0, o1, k0, k1);
  } else {
    finish<G, MODE != MODE_RECOVER_L>(a, d, Pa, acc, mtab, o0, o1, k0, k1);
  }
}

template <int P, int MODE, bool EXT = false>
__global__ void __launch_bounds__(GeoM<P, MODE>::THREADS + 32, (Layout<P, MODE>::BLOCKS)) zp_kernel(const __grid_constant__ ZpArgs a) {
  using G = GeoM<P, MODE>;
  using LY = Layout<P, MODE>;
  constexpr int C = G::C, CB = G::CB, TB = G::TB, NT = G::THREADS, ST = LY::STAGES, NOUT = LY::NOUT;
  // the combine runs the recovery epilogue on its folded partials; its tiles are counted from the
  // start of its word range (obase = range_lo), every other mode's from the start of the strip
  constexpr int EMODE = MODE == MODE_COMBINE ? MODE_RECOVER : MODE;
  const uint64_t obase = MODE == MODE_COMBINE ? a.range_lo : 0;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint8_t* outb = smem + (size_t)ST * TB;
  uint2* mtab = reinterpret_cast<uint2*>(outb + (size_t)NOUT * TB);
  uint64_t* full = reinterpret_cast<uint64_t*>(outb + (size_t)NOUT * TB + G::MTAB_BYTES);
  uint64_t* empty = full + ST;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  build_mtab<G>(mtab);
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
  // A strip length that leaves less than a tile (c1: 1 KiB of every 64 KiB strip) is finished by
  // one partial TMA tile when the kernel supports it (lane-aligned words, encode / recovery);
  // its chunks past the data compute on stale stage bytes that are never stored.
  constexpr bool PART = has_partial_tile<P, MODE, EXT>();
  auto tile_len = [&](uint64_t t) -> uint32_t {
    if constexpr (PART) return (a.last_tile != 0u && t + 1 == tiles) ? a.last_tile : static_cast<uint32_t>(TB);
    return static_cast<uint32_t>(TB);
  };

  if (warp == NT / 32) {
    // ------------------------------------------------ producer: one lane issues all TMA rows
    if (lane == 0) {
      uint32_t stage = 0, ph = 0;
      for (uint64_t it = blockIdx.x; it < body_items; it += gridDim.x) {
        const int s = static_cast<int>(it / tiles);
        const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
        const ItemDesc d = item_desc<MODE, EXT>(a, s);
        const int R = num_rows<MODE>(a, d);
        for (int r = 0; r < R; r++) {
          const uint8_t* g = in_ptr<MODE>(a, r, d, s, t * TB);
          const uint32_t len = tile_len(t);
          // the whole row tile lies inside its strip (combine: inside the slot's range)
          ZP_CHECK(t * TB + len <= (MODE == MODE_COMBINE ? a.range_hi - a.range_lo
                                                         : row_len(a, row_strip<MODE>(a, r, d))));
          ZP_CHECK((reinterpret_cast<uintptr_t>(g) & 15u) == 0 && len % 16 == 0);
          mbar_wait(&empty[stage], ph ^ 1u);
          mbar_expect_tx(&full[stage], len);
          tma_load_row(stages + (size_t)stage * TB, g, len, &full[stage]);
          if (++stage == ST) { stage = 0; ph ^= 1u; }
        }
      }
    }
    return;
  }

  // -------------------------------------------------- consumers: body tiles via the pipeline
  uint32_t stage = 0, ph = 0;
  const uint8_t* my_stages = stages + tid * CB;
  const uint32_t full_sa = smem_u32(full), empty_sa = smem_u32(empty);
  for (uint64_t it = blockIdx.x; it < body_items; it += gridDim.x) {
    const int s = static_cast<int>(it / tiles);
    const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
    const ItemDesc d = item_desc<MODE, EXT>(a, s);
    const int R = num_rows<MODE>(a, d);
    uint32_t Pa[C];
    uint32_t NEW[C];  // unused in the body path (update stages the new row in SMEM)
    Acc<G> acc;
    acc.zero();
#pragma unroll
    for (int l = 0; l < C; l++) Pa[l] = 0;
    if constexpr (MODE == MODE_UPDATE) {  // the new row goes straight to output slot 2
      if (tid == 0) bulk_wait_read0();
      named_bar_sync(1, NT);
    }
    // (words that straddle lanes; for lane-aligned words, n | 32, the generic row loop measured
    // faster: c1 encode / recovery -5 / -8 % with fold_item)
    if constexpr ((MODE == MODE_ENCODE || MODE == MODE_RECOVER || MODE == MODE_RECOVER_L) && !EXT && (32 % G::n != 0)) {
      fold_item<G, ST>(a, d, my_stages, full_sa, empty_sa, mtab, lane, stage, ph, Pa, acc);
    } else if constexpr ((MODE == MODE_ENCODE || MODE == MODE_RECOVER) && EXT && (32 % G::n != 0)) {
      fold_item_ext<G, ST>(a, d, my_stages, full_sa, empty_sa, mtab, lane, stage, ph, Pa, acc);
    } else
    for (int r = 0; r < R; r++) {
      uint32_t L[C];
      mbar_wait(&full[stage], ph);
      ld_chunk_smem<C>(stages + (size_t)stage * TB + tid * CB, L);
      if constexpr (MODE == MODE_COMBINE) {
        fold_partial<G>(r, L, Pa, acc);
      } else {
        int k = row_strip<MODE>(a, r, d);
        if constexpr (MODE == MODE_UPDATE) {
          if (k == K_NEW) {
            k = d.x;  // the new data folds in like the strip it replaces
            st_chunk_smem<C>(outb + 2 * TB + tid * CB, L);
          }
        }
        fold_row<G, EXT>(a, d, k, L, mtab, Pa, acc);
      }
      consumer_release(empty_sa + 8u * stage, lane);
      if (++stage == ST) { stage = 0; ph ^= 1u; }
    }
    uint32_t o0[C], o1[C];
    int k0 = 0, k1 = 0, k2 = 0;
    epilogue<EMODE, G, true, EXT>(a, d, s, Pa, acc, NEW, mtab, o0, o1, k0, k1, k2);
#ifdef ZP_NOOP_RECOVER  // negative control of bench.py's verification: recovery stores nothing
    if constexpr (MODE == MODE_RECOVER || MODE == MODE_RECOVER_L) continue;
#endif
    if constexpr (NOUT > 0) {
      if constexpr (MODE != MODE_UPDATE) {  // (update waited at the start of the item)
        if (tid == 0) bulk_wait_read0();  // previous item's bulk stores have read outb
        named_bar_sync(1, NT);
      }
      st_chunk_smem<C>(outb + tid * CB, o0);
      st_chunk_smem<C>(outb + TB + tid * CB, o1);
      fence_proxy_async_smem();
      named_bar_sync(1, NT);
      if (tid == 0) {
        const uint64_t ob = obase + t * TB;
        const uint32_t len = tile_len(t);
        // every stored tile lies inside its output strip (partial: inside one owner's slot)
        ZP_CHECK(ob + len <= row_len(a, k0) && ob + len <= row_len(a, k1));
        if constexpr (NOUT == 3) ZP_CHECK(ob + len <= row_len(a, k2));
        if constexpr (MODE == MODE_PARTIAL)
          ZP_CHECK(ob / a.range_bytes < static_cast<uint64_t>(a.nranges) &&
                   ob % a.range_bytes + TB <= a.range_bytes);
        tma_store_row(out_ptr(a, k0, s, ob), outb, len);
        tma_store_row(out_ptr(a, k1, s, ob), outb + TB, len);
        if constexpr (NOUT == 3) tma_store_row(out_ptr(a, k2, s, ob), outb + 2 * TB, len);
        bulk_commit();
      }
    }
  }

  // -------------------------------------------------- tail units: direct byte-precise path
  const uint64_t tups = a.tail_units_per_stripe;
  const uint64_t tail_total = tups * static_cast<uint64_t>(a.num_stripes);
  const uint64_t body_end = tiles * TB;
  // in a small launch (fewer body items than CTAs) the tail units are dealt from the LAST CTA down,
  // so the extra CTAs at the end of the grid take them at once, in parallel with the body items;
  // in a large one from the first CTA up (measured 1-2 % better there)
  const uint64_t tail_rank = gridDim.x > body_items ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
  for (uint64_t u = tail_rank * NT + tid; u < tail_total; u += static_cast<uint64_t>(gridDim.x) * NT) {
    const int s = static_cast<int>(u / tups);
    const uint64_t roff = body_end + (u - static_cast<uint64_t>(s) * tups) * CB;  // row offset
    const uint64_t off = obase + roff;                                           // strip offset
    const ItemDesc d = item_desc<MODE, EXT>(a, s);
    const int R = num_rows<MODE>(a, d);
    uint32_t Pa[C];
    uint32_t NEW[C];  // update mode only (dead otherwise)
    Acc<G> acc;
    acc.zero();
#pragma unroll
    for (int l = 0; l < C; l++) Pa[l] = 0;
#pragma unroll 1
    for (int r = 0; r < R; r++) {
      uint32_t L[C];
      if constexpr (MODE == MODE_COMBINE) {
        ld_chunk_global<C>(in_ptr<MODE>(a, r, d, s, roff), off, a.pbytes, L);
        fold_partial<G>(r, L, Pa, acc);
        continue;
      } else {
        int k = row_strip<MODE>(a, r, d);
        ld_chunk_global<C>(row_ptr(a, k, s) + off, off, row_len(a, k), L);
        if constexpr (MODE == MODE_UPDATE) {
          if (k == K_NEW) {  // old d_k (row 0) of this chunk is already folded: overwrite it now
            k = d.x;
            st_chunk_global<C>(const_cast<uint8_t*>(row_ptr(a, k, s)) + off, off, row_len(a, k), L);
          }
        }
        fold_row<G, EXT>(a, d, k, L, mtab, Pa, acc);
      }
    }
    uint32_t o0[C], o1[C];
    int k0 = 0, k1 = 0, k2 = 0;
    if constexpr (MODE == MODE_SCRUB) {  // lanes of a warp may work on different stripes here
      epilogue<MODE, G, false, EXT>(a, d, s, Pa, acc, NEW, mtab, o0, o1, k0, k1, k2);
    } else {
      epilogue<EMODE, G, true, EXT>(a, d, s, Pa, acc, NEW, mtab, o0, o1, k0, k1, k2);
#ifdef ZP_NOOP_RECOVER
      if constexpr (MODE == MODE_RECOVER || MODE == MODE_RECOVER_L) continue;
#endif
      st_chunk_global<C>(out_ptr(a, k0, s, off), off, row_len(a, k0), o0);
      st_chunk_global<C>(out_ptr(a, k1, s, off), off, row_len(a, k1), o1);
    }
  }
  if constexpr (NOUT > 0)
    if (tid == 0) bulk_wait0();
}

template <int P, int M>
void fill_geo(FastEntry& e) {
  if constexpr (M < NUM_MODES) {
    using G = GeoM<P, M>;
    e.chunk_bytes[M] = G::CB;
    e.tile_bytes[M] = G::TB;
    e.threads[M] = G::THREADS;
    e.partial_tile[M] = has_partial_tile<P, M, false>() ? 1 : 0;
    fill_geo<P, M + 1>(e);
  }
}

template <int P, bool WITH_EXT>
FastEntry make_entry() {
  FastEntry e{};
  e.p = P;
  fill_geo<P, 0>(e);
  e.kernel[MODE_ENCODE] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_ENCODE>);
  e.kernel[MODE_RECOVER] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_RECOVER>);
  e.kernel[MODE_RECOVER_L] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_RECOVER_L>);
  e.smem_bytes[MODE_RECOVER_L] = Layout<P, MODE_RECOVER_L>::SMEM;
  e.kernel[MODE_SCRUB] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_SCRUB>);
  e.kernel[MODE_UPDATE] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_UPDATE>);
  e.kernel[MODE_PARTIAL] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_PARTIAL>);
  e.smem_bytes[MODE_PARTIAL] = Layout<P, MODE_PARTIAL>::SMEM;
  e.kernel[MODE_COMBINE] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_COMBINE>);
  e.smem_bytes[MODE_COMBINE] = Layout<P, MODE_COMBINE>::SMEM;
  e.smem_bytes[MODE_ENCODE] = Layout<P, MODE_ENCODE>::SMEM;
  e.smem_bytes[MODE_RECOVER] = Layout<P, MODE_RECOVER>::SMEM;
  e.smem_bytes[MODE_SCRUB] = Layout<P, MODE_SCRUB>::SMEM;
  e.smem_bytes[MODE_UPDATE] = Layout<P, MODE_UPDATE>::SMEM;
  if constexpr (WITH_EXT) {
    e.kernel_ext[MODE_ENCODE] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_ENCODE, true>);
    e.kernel_ext[MODE_RECOVER] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_RECOVER, true>);
    e.kernel_ext[MODE_SCRUB] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_SCRUB, true>);
    e.kernel_ext[MODE_UPDATE] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_UPDATE, true>);
    e.kernel_ext[MODE_PARTIAL] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_PARTIAL, true>);
    e.smem_ext[MODE_PARTIAL] = Layout<P, MODE_PARTIAL>::SMEM;
    e.kernel_ext[MODE_COMBINE] = reinterpret_cast<const void*>(&zp_kernel<P, MODE_COMBINE, true>);
    e.smem_ext[MODE_COMBINE] = Layout<P, MODE_COMBINE>::SMEM;
    e.smem_ext[MODE_ENCODE] = Layout<P, MODE_ENCODE>::SMEM;
    e.smem_ext[MODE_RECOVER] = Layout<P, MODE_RECOVER>::SMEM;
    e.smem_ext[MODE_SCRUB] = Layout<P, MODE_SCRUB>::SMEM;
    e.smem_ext[MODE_UPDATE] = Layout<P, MODE_UPDATE>::SMEM;
  }
  return e;
}

}  // namespace zp

// Basic-code kernels for p (all four modes); WITH_EXT also instantiates the extended-code
// (Eq. (qext), N > p) kernels -- only for primes satisfying Theorem 25.3.
#define ZP_INSTANTIATE_FAST_IMPL(PP, WITH_EXT)                                               \
  namespace zp {                                                                             \
  template __global__ void zp_kernel<PP, MODE_ENCODE>(const __grid_constant__ ZpArgs);        \
  template __global__ void zp_kernel<PP, MODE_RECOVER>(const __grid_constant__ ZpArgs);       \
  template __global__ void zp_kernel<PP, MODE_RECOVER_L>(const __grid_constant__ ZpArgs);     \
  template __global__ void zp_kernel<PP, MODE_SCRUB>(const __grid_constant__ ZpArgs);         \
  template __global__ void zp_kernel<PP, MODE_UPDATE>(const __grid_constant__ ZpArgs);        \
  template __global__ void zp_kernel<PP, MODE_PARTIAL>(const __grid_constant__ ZpArgs);       \
  template __global__ void zp_kernel<PP, MODE_COMBINE>(const __grid_constant__ ZpArgs);       \
  const FastEntry* fast_entry_##PP() {                                                       \
    static const FastEntry e = make_entry<PP, WITH_EXT>();                                   \
    return &e;                                                                               \
  }                                                                                          \
  }
#define ZP_INSTANTIATE_FAST(PP) ZP_INSTANTIATE_FAST_IMPL(PP, false)
#define ZP_INSTANTIATE_FAST_EXT(PP)                                                          \
  namespace zp {                                                                             \
  template __global__ void zp_kernel<PP, MODE_ENCODE, true>(const __grid_constant__ ZpArgs);  \
  template __global__ void zp_kernel<PP, MODE_RECOVER, true>(const __grid_constant__ ZpArgs); \
  template __global__ void zp_kernel<PP, MODE_SCRUB, true>(const __grid_constant__ ZpArgs);   \
  template __global__ void zp_kernel<PP, MODE_UPDATE, true>(const __grid_constant__ ZpArgs);  \
  template __global__ void zp_kernel<PP, MODE_PARTIAL, true>(const __grid_constant__ ZpArgs); \
  template __global__ void zp_kernel<PP, MODE_COMBINE, true>(const __grid_constant__ ZpArgs); \
  }                                                                                          \
  ZP_INSTANTIATE_FAST_IMPL(PP, true)
