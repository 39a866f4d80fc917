// zp_generic.cu -- runtime-p Z_p-RAID kernel (any odd prime p <= 257) for primes without a
// compile-time specialisation (zp_fast.cuh).  Same mathematics, simpler mapping:
//   * one thread per byte-aligned group of g = 8/gcd(n,8) words (so outputs are whole bytes
//     and no two threads touch the same byte);
//   * each word is held as a p-bit value in NL = ceil(p/32) 32-bit limbs (NL is a template
//     parameter, p a runtime value; slot bit p-1 = the R' overflow), extracted from the strip
//     with funnel-shifted 32-bit reads; multiplication by x^a is a rotation of the p-bit slot
//     done limb-wise (a funnel-shift stage plus a log2(NL)-step limb barrel shifter with
//     static register indexing); the reduction pi is deferred to the end of each sum
//     (DESIGN.md "kernels");
//   * the class epilogues are the same as the fast path (Lemma 23.2 proof PAPER.md:380-401,
//     Sec. 4.6), the DD inverse by the same doubling chain.
// No TMA and no shared memory: the path for primes outside the fast set.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "zp_args.h"

namespace zp {
namespace {

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

// 32 bits of the strip starting at bit `pos` (zero past `len` bytes).
__device__ __forceinline__ uint32_t read32(const uint8_t* g, uint64_t len, uint64_t pos) {
  const uint64_t w4 = pos >> 5;
  if ((reinterpret_cast<uintptr_t>(g) & 3u) == 0 && 4 * w4 + 8 <= len) {
    const uint32_t* g4 = reinterpret_cast<const uint32_t*>(g);
    return __funnelshift_r(__ldg(g4 + w4), __ldg(g4 + w4 + 1), static_cast<uint32_t>(pos & 31));
  }
  const uint64_t b = pos >> 3;
  uint64_t v = 0;
#pragma unroll
  for (int i = 0; i < 5; i++)
    if (b + i < len) v |= static_cast<uint64_t>(__ldg(g + b + i)) << (8 * i);
  return static_cast<uint32_t>(v >> (pos & 7));
}

// Word w (n bits at stream bit w*n) of a strip of `len` bytes.
template <int NL>
__device__ __forceinline__ void load_word(const uint8_t* g, uint64_t len, uint64_t w, int n, Word<NL>& out) {
  const uint64_t b0 = w * static_cast<uint64_t>(n);
#pragma unroll
  for (int i = 0; i < NL; i++) out.v[i] = (32 * i < n && (b0 >> 3) < len) ? (read32(g, len, b0 + 32 * i) & low_mask(n, i)) : 0u;
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

__device__ Desc desc_of(const ZpArgs& a, int s, int mode, int p) {
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

constexpr int GROUP_MAX_WORDS32 = 33;  // g*n/8 <= n/2 <= 128 bytes (+1 limb of spill)

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

// buf (group bit stream) |= word v at bit offset o.
template <int NL>
__device__ __forceinline__ void put_word(uint32_t* buf, const Word<NL>& v, int o, int n) {
#pragma unroll
  for (int i = 0; i < NL; i++) {
    if (32 * i >= n) break;
    const int pos = o + 32 * i, idx = pos >> 5, sh = pos & 31;
    buf[idx] |= v.v[i] << sh;
    if (sh) buf[idx + 1] |= v.v[i] >> (32 - sh);
  }
}

template <int NL>
__global__ void zp_generic_kernel(const __grid_constant__ ZpArgs a, int p, int mode) {
  const int n = p - 1;
  const int g = 8 / (n & 7 ? ((n & 3) ? 2 : 4) : 8);  // 8 / gcd(n, 8)
  const int gbytes = g * n / 8;
  const int glimbs = (gbytes + 3) / 4;
  const uint64_t W = (8 * a.bytes + n - 1) / n;
  uint64_t g0, g1;
  group_span(a, mode, n, g, gbytes, g0, g1);
  const uint64_t groups = g1 - g0;
  const uint64_t total = groups * static_cast<uint64_t>(a.num_stripes);
  for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < total;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(u / groups);
    const uint64_t grp = g0 + (u - static_cast<uint64_t>(s) * groups);
    const Desc d = desc_of(a, s, mode, p);
    const bool ext = a.N > p;
    // rows: partial = this rank's surviving strips [k_lo, k_hi); combine = nsrc partial slots
    int R = mode == KMODE_SCRUB ? a.N + 2 : (mode == KMODE_UPDATE ? a.upd_rows : a.N);
    if (mode == KMODE_PARTIAL)
      R = a.k_hi - a.k_lo - (d.x >= a.k_lo && d.x < a.k_hi) - (d.y >= a.k_lo && d.y < a.k_hi);
    if (mode == KMODE_COMBINE) R = a.nsrc;
    int kout[3] = {0, 0, 0};
    int nout = 2;
    if (d.cls == 0) { kout[0] = a.N; kout[1] = a.N + 1; }
    else if (d.cls == 1) { kout[0] = d.x; kout[1] = a.N + 1; }
    else if (d.cls == 2) { kout[0] = d.x; kout[1] = a.N; }
    else if (d.cls == 3) { kout[0] = d.x; kout[1] = d.y; }
    else if (d.cls == 4) { nout = 0; }
    else { kout[0] = a.N; kout[1] = a.N + 1; kout[2] = d.x; nout = 3; }
    uint32_t ob[3][GROUP_MAX_WORDS32];
    for (int q = 0; q < nout; q++)
      for (int i = 0; i <= glimbs; i++) ob[q][i] = 0;
    uint32_t bad = 0;
    for (int wi = 0; wi < g; wi++) {
      const uint64_t w = grp * g + wi;
      Word<NL> Pa, acc, L, NEWW, o[3];
      wzero(Pa);
      wzero(acc);
      wzero(NEWW);
      for (int r = 0; r < R; r++) {
        if (mode == KMODE_COMBINE) {  // partial slots hold reduced words of bytes [range_lo, ...)
          const uint64_t so = static_cast<uint64_t>(s) * a.part_stride;
          const uint64_t wl = w - (a.range_lo * 8) / n, ll = a.pbytes - a.range_lo;
          load_word(a.src_p[r] + so, ll, wl, n, L);
          wxor(Pa, L);
          load_word(a.src_q[r] + so, ll, wl, n, L);
          wxor(acc, L);
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
        load_word(rptr(a, k, s), rlen(a, k), w, n, L);
        if (k == K_NEW) {
          NEWW = L;
          k = d.x;
        }
        if (k <= a.N) wxor(Pa, L);
        if (k != a.N) {
          if (ext && k < a.N) {
            add_coeff(acc, L, k, p);
          } else {
            int amt = ((k < a.N ? k : p) - d.base) % p;
            if (amt < 0) amt += p;
            rot_acc(acc, L, amt, p);
          }
        }
      }
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
        rot_acc(acc, Pa, d.x, p);
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
        int top = 31 - __clz(M);
        int m = 1;
        for (int bit = top - 1; bit >= 0; bit--) {
          Word<NL> nx = S;
          rot_acc(nx, S, (bz * m) % p, p);
          reduce(nx, p);
          S = nx;
          m *= 2;
          if ((M >> bit) & 1) {
            nx = S;
            rot_acc(nx, t, (bz * m) % p, p);
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
        bad += (w < W) && nz;
      } else {  // update
        o[0] = Pa;
        reduce(acc, p);
        o[1] = acc;
        o[2] = NEWW;
      }
      for (int q = 0; q < nout; q++) put_word(ob[q], o[q], wi * n, n);
    }
    if (mode == KMODE_SCRUB) {
      if (bad) atomicAdd(a.counts + s, bad);
      continue;
    }
    const uint64_t byte0 = grp * static_cast<uint64_t>(gbytes);
    for (int q = 0; q < nout; q++) {
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
      const int nb = static_cast<int>(left < static_cast<uint64_t>(gbytes) ? left : gbytes);
      if ((reinterpret_cast<uintptr_t>(gq) & 3u) == 0 && nb == gbytes && (gbytes & 3) == 0) {
        for (int i = 0; i < glimbs; i++) reinterpret_cast<uint32_t*>(gq)[i] = ob[q][i];
      } else {
        for (int i = 0; i < nb; i++) gq[i] = static_cast<uint8_t>(ob[q][i >> 2] >> (8 * (i & 3)));
      }
    }
  }
}

}  // namespace

cudaError_t generic_launch(const ZpArgs& a, int p, int mode, cudaStream_t st, int num_sms) {
  const int n = p - 1;
  const int g = 8 / (n & 7 ? ((n & 3) ? 2 : 4) : 8);
  const int gbytes = g * n / 8;
  const uint64_t W = (8 * a.bytes + n - 1) / n;
  uint64_t g0 = 0, g1 = (W + g - 1) / g;
  if (mode == KMODE_COMBINE) {
    g0 = a.range_lo / gbytes;
    g1 = std::min<uint64_t>(g1, (a.range_hi + gbytes - 1) / gbytes);
    if (g1 < g0) g1 = g0;
  }
  const uint64_t total = (g1 - g0) * static_cast<uint64_t>(a.num_stripes);
  const int threads = 128;
  uint64_t blocks = (total + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(num_sms) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  const dim3 grid(static_cast<unsigned>(blocks));
  switch ((p + 31) / 32) {  // 32-bit limbs per p-bit slot
    case 1: zp_generic_kernel<1><<<grid, threads, 0, st>>>(a, p, mode); break;
    case 2: zp_generic_kernel<2><<<grid, threads, 0, st>>>(a, p, mode); break;
    case 3: zp_generic_kernel<3><<<grid, threads, 0, st>>>(a, p, mode); break;
    case 4: zp_generic_kernel<4><<<grid, threads, 0, st>>>(a, p, mode); break;
    case 5: zp_generic_kernel<5><<<grid, threads, 0, st>>>(a, p, mode); break;
    case 6: zp_generic_kernel<6><<<grid, threads, 0, st>>>(a, p, mode); break;
    case 7: zp_generic_kernel<7><<<grid, threads, 0, st>>>(a, p, mode); break;
    case 8: zp_generic_kernel<8><<<grid, threads, 0, st>>>(a, p, mode); break;
    default: zp_generic_kernel<9><<<grid, threads, 0, st>>>(a, p, mode); break;
  }
  return cudaGetLastError();
}

}  // namespace zp
