#pragma once
// zp_generic.cuh -- Z_p-RAID kernel for the primes without a fast (TMA) specialisation
// (zp_fast.cuh needs a period lcm(p-1, 32) of at most 32 lanes; the other 26 odd primes <= 257
// run here).  Same mathematics, simpler mapping:
//   * one thread per byte-aligned group of g = 8/gcd(n,8) words (GB = g*n/8 bytes, so outputs
//     are whole bytes and no two threads touch the same byte); p is a template parameter, so
//     the group geometry, every word's bit offset and the limb count NL = ceil(p/32) are
//     compile-time;
//   * per strip, the group's GB bytes are read with aligned 32-bit loads (realigned by one
//     funnel shift) and the g words are cut out at compile-time offsets; each word is held as
//     a p-bit value in NL 32-bit limbs (slot bit p-1 = the R' overflow); multiplication by x^a
//     is a rotation of the p-bit slot done limb-wise (a funnel-shift stage plus a log2(NL)-step
//     limb barrel shifter with static register indexing); the reduction pi is deferred to the
//     end of each sum;
//   * the class epilogues are the same as the fast path (Lemma 23.2 proof PAPER.md:380-401,
//     Sec. 4.6), the DD inverse by the same doubling chain; outputs are
//     packed at compile-time offsets and written with aligned 32-bit stores (byte stores only
//     at the group's edges).
// Encode and recovery of the basic code (N <= p) run the TMA-staged variant
// (zp_generic_tma_kernel: the same group arithmetic fed from a shared-memory ring, outputs
// bulk-stored); the other modes, the extended code and unaligned strips use zp_generic_kernel
// (direct global loads, no shared memory).
#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <type_traits>
#include <cuda_runtime.h>

#include "tma_ring.cuh"
#include "zp_args.h"

namespace zp {
namespace gen {

template <int NL>
struct Word {
  uint32_t v[NL];
};

template <int NL>
__device__ __forceinline__ void wzero(Word<NL>& w) {
#pragma unroll
  for (int i = 0; i < NL; i++) w.v[i] = 0;
}
template <int NL>
__device__ __forceinline__ void wxor(Word<NL>& a, const Word<NL>& b) {
#pragma unroll
  for (int i = 0; i < NL; i++) a.v[i] ^= b.v[i];
}
// Mask of the low `bits` bits, limb i.
__device__ __forceinline__ uint32_t low_mask(int bits, int i) {
  const int r = bits - 32 * i;
  return r >= 32 ? 0xFFFFFFFFu : (r <= 0 ? 0u : ((1u << r) - 1u));
}

// out = in << s (s < 32*NL), bits beyond 32*NL dropped.
template <int NL>
__device__ __forceinline__ void shl(const Word<NL>& in, int s, Word<NL>& t) {
  const uint32_t r = static_cast<uint32_t>(s & 31);
  const int q = s >> 5;
#pragma unroll
  for (int i = NL - 1; i >= 0; i--) t.v[i] = __funnelshift_l(i > 0 ? in.v[i - 1] : 0u, in.v[i], r);
#pragma unroll
  for (int b = 1; b < NL; b <<= 1)
    if (q & b) {
#pragma unroll
      for (int i = NL - 1; i >= 0; i--) t.v[i] = i >= b ? t.v[i - b] : 0u;
    }
}
// out = in >> s (s < 32*NL).
template <int NL>
__device__ __forceinline__ void shr(const Word<NL>& in, int s, Word<NL>& t) {
  const uint32_t r = static_cast<uint32_t>(s & 31);
  const int q = s >> 5;
#pragma unroll
  for (int i = 0; i < NL; i++) t.v[i] = __funnelshift_r(in.v[i], i + 1 < NL ? in.v[i + 1] : 0u, r);
#pragma unroll
  for (int b = 1; b < NL; b <<= 1)
    if (q & b) {
#pragma unroll
      for (int i = 0; i < NL; i++) t.v[i] = i + b < NL ? t.v[i + b] : 0u;
    }
}

// acc ^= rot_a(src) inside the p-bit slot (src has slot bit p-1 clear; a in [0, p)):
// x^a * src in R' = F2[x]/(x^p + 1) (Eq. (powers)).
template <int NL>
__device__ __forceinline__ void rot_acc(Word<NL>& acc, const Word<NL>& src, int a, int p) {
  if (a == 0) {
    wxor(acc, src);
    return;
  }
  Word<NL> l, r;
  shl(src, a, l);
  shr(src, p - a, r);
#pragma unroll
  for (int i = 0; i < NL; i++) acc.v[i] ^= (l.v[i] | r.v[i]) & low_mask(p, i);
}

// The same rotation for a compile-time p with the whole-limb parts of both shifts dispatched to
// compile-time limb offsets: acc ^= (src << a) ^ (src >> (p - a)) limb by limb, one funnel shift
// per limb and shift instead of a funnel stage plus a log2(NL)-step select barrel (the two parts
// occupy disjoint bits [a, p) and [0, a) of the slot).  Q1 = a >> 5; Q2 = (p - a) >> 5 takes one
// of two values for a given Q1.
template <int P, int Q1, int Q2>
__device__ __forceinline__ void rot_static(Word<(P + 31) / 32>& acc, const Word<(P + 31) / 32>& src, uint32_t r1,
                                           uint32_t r2) {
  constexpr int NL = (P + 31) / 32;
#pragma unroll
  for (int i = 0; i < NL; i++) {
    const uint32_t lh = (i - Q1 >= 0 && i - Q1 < NL) ? src.v[(i - Q1 >= 0 && i - Q1 < NL) ? i - Q1 : 0] : 0u;
    const uint32_t ll = (i - Q1 - 1 >= 0 && i - Q1 - 1 < NL) ? src.v[(i - Q1 - 1 >= 0 && i - Q1 - 1 < NL) ? i - Q1 - 1 : 0] : 0u;
    const uint32_t rl = (i + Q2 < NL) ? src.v[(i + Q2 < NL) ? i + Q2 : 0] : 0u;
    const uint32_t rh = (i + Q2 + 1 < NL) ? src.v[(i + Q2 + 1 < NL) ? i + Q2 + 1 : 0] : 0u;
    const uint32_t v = __funnelshift_l(ll, lh, r1) ^ __funnelshift_r(rl, rh, r2);
    acc.v[i] ^= (32 * (i + 1) <= P) ? v : (v & low_mask(P, i));
  }
}
template <int P, int Q1>
__device__ __forceinline__ void rot_q1(Word<(P + 31) / 32>& acc, const Word<(P + 31) / 32>& src, uint32_t r1, int q2,
                                       uint32_t r2) {
  constexpr int QB = (P - 32 * Q1) >> 5;
  constexpr int QA = (P - 32 * Q1 - 31) >= 0 ? (P - 32 * Q1 - 31) >> 5 : 0;
  if constexpr (QA == QB) {
    rot_static<P, Q1, QB>(acc, src, r1, r2);
  } else {
    if (q2 == QB) rot_static<P, Q1, QB>(acc, src, r1, r2);
    else rot_static<P, Q1, QA>(acc, src, r1, r2);
  }
}
template <int P, int Q1 = 0>
__device__ __forceinline__ void rot_dispatch_q(int q1, Word<(P + 31) / 32>& acc, const Word<(P + 31) / 32>& src,
                                               uint32_t r1, int q2, uint32_t r2) {
  if constexpr (32 * Q1 < P) {
    if (q1 == Q1) {
      rot_q1<P, Q1>(acc, src, r1, q2, r2);
      return;
    }
    rot_dispatch_q<P, Q1 + 1>(q1, acc, src, r1, q2, r2);
  }
}
template <int P>
__device__ __forceinline__ void rot_acc_t(Word<(P + 31) / 32>& acc, const Word<(P + 31) / 32>& src, int a) {
  if (a == 0) {
    wxor(acc, src);
    return;
  }
  const int b = P - a;
  rot_dispatch_q<P>(a >> 5, acc, src, static_cast<uint32_t>(a & 31), b >> 5, static_cast<uint32_t>(b & 31));
}

// pi: if slot bit p-1 is set, flip bits 0..n-1 and clear bit p-1.
template <int NL>
__device__ __forceinline__ void reduce(Word<NL>& w, int p) {
  const int n = p - 1;
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < NL; i++)
    if (i == (n >> 5)) t = (w.v[i] >> (n & 31)) & 1u;  // (static register indexing)
  const uint32_t f = 0u - t;
#pragma unroll
  for (int i = 0; i < NL; i++) w.v[i] = (w.v[i] ^ (f & low_mask(n, i))) & low_mask(n, i);
}

struct Desc {
  int x, y, cls, base;  // cls: 0 PQ, 1 DQ, 2 DP, 3 DD, 4 scrub, 5 update (x = rewritten strip)
};

__device__ __forceinline__ Desc desc_of(const ZpArgs& a, int s, int mode, int p) {
  Desc d;
  if (mode == KMODE_SCRUB) {
    d.x = d.y = -1; d.cls = 4; d.base = 0;
    return d;
  }
  if (mode == KMODE_UPDATE) {
    d.x = a.upd ? a.upd[static_cast<int64_t>(s) * a.upd_stride] : a.upd_k;
    d.y = -1; d.cls = 5; d.base = 0;
    return d;
  }
  int i = a.N, j = a.N + 1;
  if (mode == KMODE_RECOVER || mode == KMODE_PARTIAL || mode == KMODE_COMBINE) {
    if (a.er) {
      const int2 e = a.er[static_cast<int64_t>(s) * a.er_stride];
      i = e.x; j = e.y;
    } else {
      i = a.ei; j = a.ej;
    }
  }
  d.x = i < j ? i : j;
  d.y = i < j ? j : i;
  if (d.y == a.N + 1) d.cls = (d.x == a.N) ? 0 : 1;  // PQ : DQ
  else d.cls = (d.y == a.N) ? 2 : 3;                  // DP : DD
  // basic code: rotation origin at the lost strip; extended code (N > p): origin 0 + ExtProg
  d.base = (a.N <= p && (d.cls == 2 || d.cls == 3)) ? d.x : 0;
  return d;
}

// acc ^= g_k * v with g_k the Eq. (qext) coefficient of data strip k (x^k, or 1 + x^{k-p+1}).
template <int NL>
__device__ __forceinline__ void add_coeff(Word<NL>& acc, const Word<NL>& v, int k, int p) {
  if (k < p) {
    rot_acc(acc, v, k, p);
  } else {
    rot_acc(acc, v, 0, p);
    rot_acc(acc, v, k - p + 1, p);
  }
}

// out = u * t for the pair's ExtProg: u = sum_i x^{e_i}, or, for a geometric pair,
// u = x^{e0} sum_{m<(p+1)/2} x^{bz m} (= x^{e0} (1 + x^{bz/2})^{-1}, reading R11).
template <int NL>
__device__ void mul_prog(const Word<NL>& t, const ExtProg* pr, int p, Word<NL>& out) {
  wzero(out);
  if (pr->geo_bz) {
    for (int m = 0; m < (p + 1) / 2; m++) rot_acc(out, t, (pr->geo_bz * m + pr->geo_e0) % p, p);
  } else {
    for (int i = 0; i < pr->nu; i++) rot_acc(out, t, pr->e[i], p);
  }
  reduce(out, p);
}

__device__ __forceinline__ uint64_t sstride(const ZpArgs& a, int k) { return k < a.N ? a.data_stride : a.parity_stride; }
constexpr int K_NEW = -1;
__device__ __forceinline__ const uint8_t* rptr(const ZpArgs& a, int k, int s) {
  return k == K_NEW ? a.nbase + static_cast<uint64_t>(s) * a.new_stride : a.base[k] + static_cast<uint64_t>(s) * sstride(a, k);
}
__device__ __forceinline__ uint64_t rlen(const ZpArgs& a, int k) {
  return (k == K_NEW || k < a.N) ? a.bytes : a.pbytes;
}

// Compile-time group geometry of prime P.
template <int P>
struct GP {
  static constexpr int n = P - 1;
  static constexpr int NL = (P + 31) / 32;                                  // limbs per p-bit slot
  static constexpr int g = 8 / ((n & 7) == 0 ? 8 : ((n & 3) == 0 ? 4 : 2));  // words per group
  static constexpr int GB = g * n / 8;                                      // bytes per group
  static constexpr int W4 = (GB + 3) / 4;                                   // 32-bit words per group
  // CTAs of 128 threads per SM: 4 (<= 128 registers) while the g words x NL limbs of the two
  // accumulators fit without spilling, else 3 (measured: p = 67, 127, 181 +25-50 % at 4 vs one
  // unconstrained CTA; p = 251 spills 1.1 KB at 4 and runs best at 3)
  static constexpr int MINB = NL * g <= 20 ? 4 : 3;
};

// Group range of one launch: all groups of the strip, or (combine) the groups of bytes
// [range_lo, range_hi) -- range_lo is a multiple of the group size (host-checked).
__device__ __forceinline__ void group_span(const ZpArgs& a, int mode, int n, int g, int gbytes, uint64_t& g0,
                                           uint64_t& g1) {
  const uint64_t W = (8 * a.bytes + n - 1) / n;
  const uint64_t groups = (W + g - 1) / g;
  g0 = 0;
  g1 = groups;
  if (mode == KMODE_COMBINE) {
    g0 = a.range_lo / gbytes;
    const uint64_t e = (a.range_hi + gbytes - 1) / gbytes;
    g1 = e < groups ? e : groups;
    if (g1 < g0) g1 = g0;
  }
}

// buf[0..W4) = bytes [byte0, byte0 + 4*W4) of a row of `len` bytes, zero past `len`
// (reading R5's zero extension); buf[W4] = 0.
template <int W4>
__device__ __forceinline__ void load_group(const uint8_t* row, uint64_t len, uint64_t byte0, uint32_t (&buf)[W4 + 1]) {
  const uint8_t* pg = row + byte0;
  const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(pg) & 3u);
  buf[W4] = 0u;
  if (byte0 + 4 * W4 + 4 <= len + mis) {  // the aligned words [pg - mis, pg - mis + 4(W4+1)) lie in the row
    const uint32_t* q = reinterpret_cast<const uint32_t*>(pg - mis);
    uint32_t raw[W4 + 1];
#pragma unroll
    for (int i = 0; i <= W4; i++) raw[i] = __ldg(q + i);
#pragma unroll
    for (int i = 0; i < W4; i++) buf[i] = __funnelshift_r(raw[i], raw[i + 1], 8 * mis);
    return;
  }
#pragma unroll
  for (int i = 0; i < W4; i++) {
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; b++)
      if (byte0 + 4 * i + b < len) v |= static_cast<uint32_t>(__ldg(pg + 4 * i + b)) << (8 * b);
    buf[i] = v;
  }
}

// Word WI of the group (bits [WI*n, WI*n + n) of buf), compile-time offsets.
template <int P, int WI>
__device__ __forceinline__ void group_word(const uint32_t (&buf)[GP<P>::W4 + 1], Word<GP<P>::NL>& out) {
  constexpr int n = GP<P>::n;
#pragma unroll
  for (int i = 0; i < GP<P>::NL; i++) {
    const int pos = WI * n + 32 * i, idx = pos >> 5, sh = pos & 31;
    const uint32_t lo = idx < GP<P>::W4 + 1 ? buf[idx < GP<P>::W4 + 1 ? idx : 0] : 0u;
    const uint32_t hi = idx + 1 < GP<P>::W4 + 1 ? buf[idx + 1 < GP<P>::W4 + 1 ? idx + 1 : 0] : 0u;
    out.v[i] = 32 * i < n ? (__funnelshift_r(lo, hi, sh) & low_mask(n, i)) : 0u;
  }
}

// ob |= word v at bit offset WI*n (compile-time).
template <int P, int WI>
__device__ __forceinline__ void group_put(uint32_t (&ob)[GP<P>::W4 + 1], const Word<GP<P>::NL>& v) {
  constexpr int n = GP<P>::n;
#pragma unroll
  for (int i = 0; i < GP<P>::NL; i++) {
    if (32 * i >= n) break;
    const int pos = WI * n + 32 * i, idx = pos >> 5, sh = pos & 31;
    if (idx < GP<P>::W4 + 1) ob[idx < GP<P>::W4 + 1 ? idx : 0] |= v.v[i] << sh;
    if (sh && idx + 1 < GP<P>::W4 + 1) ob[idx + 1 < GP<P>::W4 + 1 ? idx + 1 : 0] |= v.v[i] >> (32 - sh);
  }
}

// Bytes [0, nb) of the group buffer to dst: aligned 32-bit stores, byte stores at the edges.
template <int W4>
__device__ __forceinline__ void store_group(uint8_t* dst, int nb, const uint32_t (&ob)[W4 + 1]) {
  const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 3u);
  uint32_t* q = reinterpret_cast<uint32_t*>(dst - mis);
#pragma unroll
  for (int j = 0; j <= W4; j++) {  // word j of q holds group bytes [4j - mis, 4j - mis + 4)
    const uint32_t v = __funnelshift_l(j > 0 ? ob[j > 0 ? j - 1 : 0] : 0u, ob[j], 8 * mis);
    const int b0 = 4 * j - static_cast<int>(mis);
    if (b0 >= 0 && b0 + 4 <= nb) {
      q[j] = v;
    } else {
#pragma unroll
      for (int b = 0; b < 4; b++)
        if (b0 + b >= 0 && b0 + b < nb) dst[b0 + b] = static_cast<uint8_t>(v >> (8 * b));
    }
  }
}

// Class epilogue of one word: o[0..nout) from the folded Pa / acc.
template <int P, int NL = (P + 31) / 32>
__device__ __forceinline__ void finish_word(const ZpArgs& a, const Desc& d, int mode, bool ext, Word<NL>& Pa,
                                            Word<NL>& acc, Word<NL> (&o)[2], bool valid, uint32_t& bad) {
  constexpr int p = P;
  const ExtProg* pr = ext ? a.prog + pair_index(d.x, d.y, a.N) : nullptr;
  if (mode == KMODE_PARTIAL) {  // unsolved partial syndromes (NEXT-4)
    o[0] = Pa;
    reduce(acc, p);
    o[1] = acc;
  } else if (ext && (d.cls == 1 || d.cls == 2 || d.cls == 3)) {  // extended code (Lemma 23.2 with Eq. (qext))
    if (d.cls == 1) {
      o[0] = Pa;
      add_coeff(acc, Pa, d.x, p);
      reduce(acc, p);
      o[1] = acc;
    } else if (d.cls == 2) {
      reduce(acc, p);
      mul_prog(acc, pr, p, o[0]);
      o[1] = Pa;
      wxor(o[1], o[0]);
    } else {
      add_coeff(acc, Pa, d.x, p);
      reduce(acc, p);
      mul_prog(acc, pr, p, o[1]);
      o[0] = o[1];
      wxor(o[0], Pa);
    }
  } else if (d.cls == 0) {
    o[0] = Pa;
    reduce(acc, p);
    o[1] = acc;
  } else if (d.cls == 1) {
    o[0] = Pa;
    rot_acc_t<P>(acc, Pa, d.x);
    reduce(acc, p);
    o[1] = acc;
  } else if (d.cls == 2) {
    reduce(acc, p);
    o[0] = acc;
    o[1] = Pa;
    wxor(o[1], o[0]);
  } else if (d.cls == 3) {
    wxor(acc, Pa);
    reduce(acc, p);
    const Word<NL> t = acc;
    Word<NL> S = t;
    const int M = (p + 1) / 2;
    const int bz = (2 * (d.y - d.x)) % p;
    const int top = 31 - __clz(M);
    int m = 1;
#pragma unroll 1
    for (int bit = top - 1; bit >= 0; bit--) {
      Word<NL> nx = S;
      rot_acc_t<P>(nx, S, (bz * m) % p);
      reduce(nx, p);
      S = nx;
      m *= 2;
      if ((M >> bit) & 1) {
        nx = S;
        rot_acc_t<P>(nx, t, (bz * m) % p);
        reduce(nx, p);
        S = nx;
        m += 1;
      }
    }
    o[1] = S;
    o[0] = S;
    wxor(o[0], Pa);
  } else if (d.cls == 4) {  // scrub: syndromes of both parity equations
    reduce(acc, p);
    wxor(acc, Pa);
    uint32_t nz = 0;
#pragma unroll
    for (int j = 0; j < NL; j++) nz |= acc.v[j] | Pa.v[j];
    bad += valid && nz;
  } else {  // update (the new data bytes were stored when read)
    o[0] = Pa;
    reduce(acc, p);
    o[1] = acc;
  }
}

// Output strips of a class (update: P, Q -- d_k was stored with its row; scrub: none).
__device__ __forceinline__ void out_strips(const ZpArgs& a, const Desc& d, int (&kout)[2], int& nout) {
  if (d.cls == 0) { kout[0] = a.N; kout[1] = a.N + 1; }
  else if (d.cls == 1) { kout[0] = d.x; kout[1] = a.N + 1; }
  else if (d.cls == 2) { kout[0] = d.x; kout[1] = a.N; }
  else if (d.cls == 3) { kout[0] = d.x; kout[1] = d.y; }
  else if (d.cls == 4) { nout = 0; }
  else { kout[0] = a.N; kout[1] = a.N + 1; }
}

template <int P, int WI>
struct GroupWords {  // compile-time loop over the group's words
  template <class F>
  __device__ __forceinline__ static void run(F&& f) {
    if constexpr (WI < GP<P>::g) {
      f(std::integral_constant<int, WI>{});
      GroupWords<P, WI + 1>::run(f);
    }
  }
};

// One group (g words) of stripe s through the direct path: aligned 32-bit global loads of each
// row, fold, class epilogue, aligned stores (byte stores at the group's edges).
template <int P>
__device__ __forceinline__ void group_direct(const ZpArgs& a, int mode, int s, uint64_t grp, uint64_t W) {
  using GG = GP<P>;
  constexpr int NL = GG::NL, g = GG::g, GB = GG::GB, W4 = GG::W4;
  const uint64_t byte0 = grp * static_cast<uint64_t>(GB);
  const Desc d = desc_of(a, s, mode, P);
  const bool ext = a.N > P;
  // rows: partial = this rank's surviving strips [k_lo, k_hi); combine = nsrc partial slots
  int R = mode == KMODE_SCRUB ? a.N + 2 : (mode == KMODE_UPDATE ? a.upd_rows : a.N);
  if (mode == KMODE_PARTIAL)
    R = a.k_hi - a.k_lo - (d.x >= a.k_lo && d.x < a.k_hi) - (d.y >= a.k_lo && d.y < a.k_hi);
  if (mode == KMODE_COMBINE) R = a.nsrc;
  Word<NL> Pa[g], acc[g];
#pragma unroll
  for (int wi = 0; wi < g; wi++) {
    wzero(Pa[wi]);
    wzero(acc[wi]);
  }
  uint32_t buf[W4 + 1];
  for (int r = 0; r < R; r++) {
    if (mode == KMODE_COMBINE) {  // partial slots hold reduced words of bytes [range_lo, ...)
      const uint64_t so = static_cast<uint64_t>(s) * a.part_stride;
      const uint64_t off = byte0 - a.range_lo, ll = a.pbytes - a.range_lo;
      load_group<W4>(a.src_p[r] + so, ll, off, buf);
      GroupWords<P, 0>::run([&](auto wc) {
        Word<NL> L;
        group_word<P, decltype(wc)::value>(buf, L);
        wxor(Pa[decltype(wc)::value], L);
      });
      load_group<W4>(a.src_q[r] + so, ll, off, buf);
      GroupWords<P, 0>::run([&](auto wc) {
        Word<NL> L;
        group_word<P, decltype(wc)::value>(buf, L);
        wxor(acc[decltype(wc)::value], L);
      });
      continue;
    }
    int k;
    if (mode == KMODE_SCRUB) k = r;
    else if (mode == KMODE_UPDATE) k = r == 0 ? d.x : (r == 1 ? K_NEW : a.N + r - 2);
    else {
      k = mode == KMODE_PARTIAL ? a.k_lo + r : r;
      const int lo = mode == KMODE_PARTIAL ? a.k_lo : 0;
      if (d.x >= lo && k >= d.x) k++;
      if (d.y >= lo && k >= d.y) k++;
    }
    load_group<W4>(rptr(a, k, s), rlen(a, k), byte0, buf);
    if (k == K_NEW) {
      // update: the new bytes go straight to the rewritten strip (this group's bytes of it were
      // read as row 0; bytes of neighbouring groups that the aligned loads touch are masked off)
      const uint64_t left = a.bytes > byte0 ? a.bytes - byte0 : 0;
      store_group<W4>(const_cast<uint8_t*>(rptr(a, d.x, s)) + byte0,
                      static_cast<int>(left < static_cast<uint64_t>(GB) ? left : GB), buf);
      k = d.x;
    }
    int amt = 0;
    if (!(ext && k < a.N)) {
      amt = ((k < a.N ? k : P) - d.base) % P;
      if (amt < 0) amt += P;
    }
    GroupWords<P, 0>::run([&](auto wc) {
      constexpr int WI = decltype(wc)::value;
      Word<NL> L;
      group_word<P, WI>(buf, L);
      if (k <= a.N) wxor(Pa[WI], L);
      if (k != a.N) {
        if (ext && k < a.N) add_coeff(acc[WI], L, k, P);
        else rot_acc_t<P>(acc[WI], L, amt);
      }
    });
  }
  int kout[2] = {0, 0};
  int nout = 2;
  out_strips(a, d, kout, nout);
  uint32_t ob[2][W4 + 1];
#pragma unroll
  for (int q = 0; q < 2; q++)
#pragma unroll
    for (int i = 0; i <= W4; i++) ob[q][i] = 0;
  uint32_t bad = 0;
  GroupWords<P, 0>::run([&](auto wc) {
    constexpr int WI = decltype(wc)::value;
    Word<NL> o[2];
    finish_word<P>(a, d, mode, ext, Pa[WI], acc[WI], o, grp * g + WI < W, bad);
#pragma unroll
    for (int q = 0; q < 2; q++)
      if (q < nout) group_put<P, WI>(ob[q], o[q]);
  });
  if (mode == KMODE_SCRUB) {
    if (bad) atomicAdd(a.counts + s, bad);
    return;
  }
#pragma unroll
  for (int q = 0; q < 2; q++) {
    if (q >= nout) break;
    uint8_t* gq;  // address of byte byte0 of output q
    uint64_t left;
    if (mode == KMODE_PARTIAL) {  // slot of the owner of this word range
      const int own = static_cast<int>(byte0 / a.range_bytes);
      gq = (q == 0 ? a.part_p[own] : a.part_q[own]) + static_cast<uint64_t>(s) * a.part_stride +
           (byte0 - static_cast<uint64_t>(own) * a.range_bytes);
      left = a.pbytes > byte0 ? a.pbytes - byte0 : 0;
    } else {
      gq = const_cast<uint8_t*>(rptr(a, kout[q], s)) + byte0;
      const uint64_t len = rlen(a, kout[q]);
      left = len > byte0 ? len - byte0 : 0;
    }
    const int nb = static_cast<int>(left < static_cast<uint64_t>(GB) ? left : GB);
    store_group<W4>(gq, nb, ob[q]);
  }
}

template <int P>
__global__ void __launch_bounds__(128, GP<P>::MINB) zp_generic_kernel(const __grid_constant__ ZpArgs a, int mode) {
  using GG = GP<P>;
  const uint64_t W = (8 * a.bytes + GG::n - 1) / GG::n;
  uint64_t g0, g1;
  group_span(a, mode, GG::n, GG::g, GG::GB, g0, g1);
  const uint64_t groups = g1 - g0;
  const uint64_t total = groups * static_cast<uint64_t>(a.num_stripes);
  for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < total;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(u / groups);
    group_direct<P>(a, mode, s, g0 + (u - static_cast<uint64_t>(s) * groups), W);
  }
}

// ---------------------------------------------------------------- TMA-staged encode / recovery
// The same group arithmetic fed from a TMA ring (the fast kernel's producer/consumer scheme,
// tma_ring.cuh): a tile = 128 consecutive groups of one stripe (TB = 128 * GB bytes, a multiple
// of 16); one producer lane streams the tile rows of the N surviving strips HBM -> SMEM with
// cp.async.bulk; consumer thread t reads group t of each row from SMEM (aligned 32-bit loads,
// one funnel shift), folds it, runs the class epilogue, packs the outputs into two SMEM output
// tiles, and thread 0 bulk-stores them.  The groups past the last whole tile (and every group
// when a strip is not 16-byte aligned) go through group_direct.  Basic code (N <= p), encode and
// recovery only; the other modes and the extended code keep zp_generic_kernel.
template <int P>
struct GT {
  using GG = GP<P>;
  // consumer threads = groups per tile: 256 (2 CTAs, 18 warps per SM) while a group's g words of
  // NL limbs stay at most 28 accumulator limbs, else 128 (3 CTAs; 2 from 20 limbs up).  Measured
  // (c2 shape, 256 vs 128 threads): p = 67 ... 107 +10-20 % encode and recovery, p = 127 ... 163
  // +4-17 % / +10-33 %, p = 211 (28 limbs) encode -4 %, recovery +19 %; p = 251 (32 limbs, spills)
  // -30 %; 192 threads (14 warps) lose to both
  static constexpr int NT = GG::NL * GG::g <= 28 ? 256 : 128;
  static constexpr int TB = NT * GG::GB;          // tile bytes
  static constexpr int MINB = NT >= 192 ? 2 : (GG::NL * GG::g <= 20 ? 3 : 2);  // CTAs per SM
  static constexpr int BUDGET = (227 * 1024) / MINB - 1024;
  static constexpr int ST_RAW = (BUDGET - 2 * TB - 128) / TB;
  static constexpr int ST = ST_RAW < 2 ? 2 : (ST_RAW > 8 ? 8 : ST_RAW);
  static constexpr size_t SMEM = static_cast<size_t>(ST + 2) * TB + 2 * ST * 8 + 16;
  static_assert(TB % 16 == 0, "TMA rows are multiples of 16 bytes");
  static_assert(SMEM + 1024 <= 227 * 1024 / MINB + 1024, "MINB CTAs must fit the SM's shared memory");
};

template <int P, int MODE>
__global__ void __launch_bounds__(GT<P>::NT + 32, GT<P>::MINB) zp_generic_tma_kernel(const __grid_constant__ ZpArgs a) {
  using GG = GP<P>;
  using T = GT<P>;
  constexpr int NL = GG::NL, g = GG::g, GB = GG::GB, W4 = GG::W4, NT = T::NT, TB = T::TB, ST = T::ST;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint8_t* outb = smem + static_cast<size_t>(ST) * TB;
  // (one 16-byte pad after the output tiles: the last group's aligned loads may read a word past
  // its stage, never past the allocation)
  uint64_t* full = reinterpret_cast<uint64_t*>(outb + 2 * static_cast<size_t>(TB) + 16);
  uint64_t* empty = full + ST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < ST; i++) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t tiles = a.body_tiles;
  const uint64_t items = tiles * static_cast<uint64_t>(a.num_stripes);
  if (warp == NT / 32) {  // producer: one lane issues every row of every item
    if (lane == 0) {
      uint32_t stage = 0, ph = 0;
      for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int s = static_cast<int>(it / tiles);
        const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
        const Desc d = desc_of(a, s, MODE, P);
        for (int r = 0; r < a.N; r++) {
          int k = r;
          if (k >= d.x) k++;
          if (k >= d.y) k++;
          mbar_wait(&empty[stage], ph ^ 1u);
          mbar_expect_tx(&full[stage], TB);
          tma_load_row(stages + static_cast<size_t>(stage) * TB, rptr(a, k, s) + t * TB, TB, &full[stage]);
          if (++stage == ST) { stage = 0; ph ^= 1u; }
        }
      }
    }
    return;
  }
  const uint32_t full_sa = smem_u32(full), empty_sa = smem_u32(empty);
  uint32_t stage = 0, ph = 0;
  const uint32_t mis = static_cast<uint32_t>(tid * GB) & 3u;
  const uint32_t* my = reinterpret_cast<const uint32_t*>(stages + (tid * GB - mis));
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int s = static_cast<int>(it / tiles);
    const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
    const Desc d = desc_of(a, s, MODE, P);
    Word<NL> Pa[g], acc[g];
#pragma unroll
    for (int wi = 0; wi < g; wi++) {
      wzero(Pa[wi]);
      wzero(acc[wi]);
    }
    for (int r = 0; r < a.N; r++) {
      int k = r;
      if (k >= d.x) k++;
      if (k >= d.y) k++;
      mbar_wait_sa(full_sa + 8u * stage, ph);
      const uint32_t* q = my + static_cast<size_t>(stage) * (TB / 4);
      uint32_t raw[W4 + 1], buf[W4 + 1];
#pragma unroll
      for (int i = 0; i <= W4; i++) raw[i] = q[i];
#pragma unroll
      for (int i = 0; i < W4; i++) buf[i] = __funnelshift_r(raw[i], raw[i + 1], 8 * mis);
      buf[W4] = 0u;
      int amt = ((k < a.N ? k : P) - d.base) % P;
      if (amt < 0) amt += P;
      GroupWords<P, 0>::run([&](auto wc) {
        constexpr int WI = decltype(wc)::value;
        Word<NL> L;
        group_word<P, WI>(buf, L);
        if (k <= a.N) wxor(Pa[WI], L);
        if (k != a.N) rot_acc_t<P>(acc[WI], L, amt);
      });
      consumer_release(empty_sa + 8u * stage, lane);
      if (++stage == ST) { stage = 0; ph ^= 1u; }
    }
    int kout[2] = {0, 0};
    int nout = 2;
    out_strips(a, d, kout, nout);
    uint32_t ob[2][W4 + 1];
#pragma unroll
    for (int q = 0; q < 2; q++)
#pragma unroll
      for (int i = 0; i <= W4; i++) ob[q][i] = 0;
    uint32_t bad = 0;
    GroupWords<P, 0>::run([&](auto wc) {
      constexpr int WI = decltype(wc)::value;
      Word<NL> o[2];
      finish_word<P>(a, d, MODE, false, Pa[WI], acc[WI], o, true, bad);
      group_put<P, WI>(ob[0], o[0]);
      group_put<P, WI>(ob[1], o[1]);
    });
    if (tid == 0) bulk_wait_read0();  // the previous item's bulk stores have read the tiles
    named_bar_sync(1, NT);
    store_group<W4>(outb + tid * GB, GB, ob[0]);
    store_group<W4>(outb + TB + tid * GB, GB, ob[1]);
    fence_proxy_async_smem();
    named_bar_sync(1, NT);
    if (tid == 0) {
      tma_store_row(const_cast<uint8_t*>(rptr(a, kout[0], s)) + t * TB, outb, TB);
      tma_store_row(const_cast<uint8_t*>(rptr(a, kout[1], s)) + t * TB, outb + TB, TB);
      bulk_commit();
    }
  }
  // groups past the body tiles: direct path, one group per consumer thread
  const uint64_t W = (8 * a.bytes + GG::n - 1) / GG::n;
  const uint64_t groups = (W + g - 1) / g;
  const uint64_t gbody = tiles * NT;
  const uint64_t tail = groups > gbody ? groups - gbody : 0;
  const uint64_t total = tail * static_cast<uint64_t>(a.num_stripes);
  for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * NT + tid; u < total; u += static_cast<uint64_t>(gridDim.x) * NT) {
    const int s = static_cast<int>(u / tail);
    group_direct<P>(a, MODE, s, gbody + (u - static_cast<uint64_t>(s) * tail), W);
  }
  if (tid == 0) bulk_wait0();
}

// CTAs per SM of a TMA kernel on the current device (dynamic shared memory attribute set once
// per device and kernel).
inline cudaError_t tma_occupancy(const void* fn, size_t smem, int threads, int* occ) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, fn);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *occ = it->second;
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int o = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (o < 1) o = 1;
  cache[key] = o;
  *occ = o;
  return cudaSuccess;
}

template <int P>
cudaError_t launch_p(const ZpArgs& a, int mode, cudaStream_t st, int num_sms) {
  using GG = GP<P>;
  // (3, 7, 31, 73 reach this kernel only with the extended code)
  if constexpr (!(P == 3 || P == 7 || P == 31 || P == 73)) {
    using T = GT<P>;
    if ((mode == KMODE_ENCODE || mode == KMODE_RECOVER) && a.N <= P && a.bytes >= static_cast<uint64_t>(T::TB)) {
      bool aligned = true;
      for (int k = 0; k < a.N + 2; k++) aligned &= (reinterpret_cast<uintptr_t>(a.base[k]) & 15u) == 0;
      if (a.num_stripes > 1) aligned &= (a.data_stride % 16 == 0) && (a.parity_stride % 16 == 0);
      if (aligned) {
        ZpArgs b = a;
        b.body_tiles = a.bytes / T::TB;
        const void* fn = mode == KMODE_ENCODE ? reinterpret_cast<const void*>(&zp_generic_tma_kernel<P, KMODE_ENCODE>)
                                              : reinterpret_cast<const void*>(&zp_generic_tma_kernel<P, KMODE_RECOVER>);
        int occ = 1;
        cudaError_t e = tma_occupancy(fn, T::SMEM, T::NT + 32, &occ);
        if (e != cudaSuccess) return e;
        const uint64_t W = (8 * a.bytes + GG::n - 1) / GG::n;
        const uint64_t groups = (W + GG::g - 1) / GG::g;
        const uint64_t tail = groups - b.body_tiles * T::NT;
        const uint64_t items = b.body_tiles * static_cast<uint64_t>(a.num_stripes);
        const uint64_t tail_ctas = (tail * static_cast<uint64_t>(a.num_stripes) + T::NT - 1) / T::NT;
        const uint64_t cap = static_cast<uint64_t>(num_sms) * occ;
        uint64_t grid = std::min<uint64_t>(cap, std::max<uint64_t>(items, tail_ctas));
        if (grid == 0) grid = 1;
        void* args[] = {&b};
        e = cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(T::NT + 32), args, T::SMEM, st);
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
      }
    }
  }
  uint64_t g0 = 0, g1 = ((8 * a.bytes + GG::n - 1) / GG::n + GG::g - 1) / GG::g;
  if (mode == KMODE_COMBINE) {
    g0 = a.range_lo / GG::GB;
    g1 = std::min<uint64_t>(g1, (a.range_hi + GG::GB - 1) / GG::GB);
    if (g1 < g0) g1 = g0;
  }
  const uint64_t total = (g1 - g0) * static_cast<uint64_t>(a.num_stripes);
  const int threads = 128;
  uint64_t blocks = (total + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(num_sms) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  zp_generic_kernel<P><<<dim3(static_cast<unsigned>(blocks)), threads, 0, st>>>(a, mode);
  return cudaGetLastError();
}

}  // namespace gen
}  // namespace zp
