// rs.cu -- NEXT-3: the paper's comparison system, Reed-Solomon RAID-6 over GF(2^8) ("DP-RAID",
// Sec. 4.1-4.4), on the same B200 pipeline as the Z_p kernels, so that the
// paper's relative claim (Z_p vs RS) can be restated on B200.
//   P = sum D_i,  Q = sum g^i D_i,  g = {02}, reduction polynomial 0x11D   (Eq. (rsparity))
//   multiplication by g on four bytes at once (SWAR form of PAPER.md:883):
//       mul2(v) = ((v & 0x7f7f7f7f) << 1) ^ (((v >> 7) & 0x01010101) * 0x1d)
//   Q by Horner's rule over the data strips in descending order; lost strips
//   are skipped by extra multiplications by g.  Recovery: Sec. 4.3 (A, B computed once per pair
//   from exp/log tables), products by a constant c as the bit-serial sum
//   sum_i c_i g^i v (no lookup tables on the data path).
#include <cstdint>
#include <cuda_runtime.h>

#include "zp_fast.cuh"  // PTX helpers, chunk I/O, ZpArgs

namespace zp {
namespace rs {

constexpr int C = 12;           // 32-bit lanes per thread-chunk (48 B: conflict-free LDS.128)
constexpr int CB = 4 * C;
constexpr int THREADS = 256;
constexpr int TB = THREADS * CB;  // 12288-byte TMA rows
// CTAs per SM and TMA stages per kernel (the Z_p kernels' occupancy rule, applied alike so the
// comparison stays like for like): encode three CTAs x 3 stages, recovery two CTAs x 7 stages.
#ifndef RS_ENC_MINB
#define RS_ENC_MINB 3
#endif
template <bool RECOVER>
struct Cfg {
  static constexpr int MINB = RECOVER ? 2 : RS_ENC_MINB;
  static constexpr int STAGES = MINB == 3 ? 3 : 7;
  static constexpr size_t SMEM = (size_t)(STAGES + 2) * TB + 512 + 2 * STAGES * 8;
};

__device__ __forceinline__ uint32_t mul2(uint32_t v) {
  return ((v & 0x7f7f7f7fu) << 1) ^ (((v >> 7) & 0x01010101u) * 0x1du);
}

template <int K>
__device__ __forceinline__ void mul2_n(uint32_t (&v)[K], int times) {
#pragma unroll 1
  for (int t = 0; t < times; t++)
#pragma unroll
    for (int l = 0; l < K; l++) v[l] = mul2(v[l]);
}

// out = c * v on every byte (bit-serial: sum over the bits i of c of g^i v).
__device__ __forceinline__ void mulc(const uint32_t (&v)[C], uint32_t c, uint32_t (&out)[C]) {
  uint32_t w[C];
#pragma unroll
  for (int l = 0; l < C; l++) { w[l] = v[l]; out[l] = 0; }
#pragma unroll 1
  for (int i = 0; i < 8; i++) {
    if ((c >> i) & 1u) {
#pragma unroll
      for (int l = 0; l < C; l++) out[l] ^= w[l];
    }
#pragma unroll
    for (int l = 0; l < C; l++) w[l] = mul2(w[l]);
  }
}

struct Desc {
  int x, y, cls;  // cls: 0 PQ, 1 DQ, 2 DP, 3 DD
};

template <bool RECOVER>
__device__ __forceinline__ Desc desc_of(const ZpArgs& a, int s) {
  int i = a.N, j = a.N + 1;
  if constexpr (RECOVER) {
    if (a.er) {
      const int2 e = a.er[static_cast<int64_t>(s) * a.er_stride];
      i = e.x; j = e.y;
    } else {
      i = a.ei; j = a.ej;
    }
  }
  Desc d;
  d.x = i < j ? i : j;
  d.y = i < j ? j : i;
  if (d.y == a.N + 1) d.cls = (d.x == a.N) ? 0 : 1;
  else d.cls = (d.y == a.N) ? 2 : 3;
  return d;
}

// Row r of an item: surviving data strips in descending order, then P, then Q.
__device__ __forceinline__ int row_strip(const ZpArgs& a, int r, const Desc& d) {
  int nd = a.N - (d.x < a.N) - (d.y < a.N);  // surviving data strips
  if (r < nd) {  // r-th survivor from the top: skip the lost data indices at or above it
    int k = a.N - 1 - r;
    if (d.y < a.N && d.y >= k) k--;
    if (d.x < a.N && d.x >= k) k--;
    return k;
  }
  r -= nd;
  if (d.x != a.N && d.y != a.N) {
    if (r == 0) return a.N;
    r--;
  }
  return a.N + 1;
}

__device__ __forceinline__ const uint8_t* rptr(const ZpArgs& a, int k, int s) {
  return a.base[k] + static_cast<uint64_t>(s) * (k < a.N ? a.data_stride : a.parity_stride);
}

struct State {
  uint32_t Pa[C], Qa[C], acc[C];
  int prev;
};

__device__ __forceinline__ void state_init(State& st, int N) {
#pragma unroll
  for (int l = 0; l < C; l++) { st.Pa[l] = 0; st.Qa[l] = 0; st.acc[l] = 0; }
  st.prev = N;
}

__device__ __forceinline__ void fold(State& st, const ZpArgs& a, int k, const uint32_t (&L)[C]) {
  if (k < a.N) {  // Horner step: acc = g^{prev-k} acc + D_k
    mul2_n<C>(st.acc, st.prev - k);
#pragma unroll
    for (int l = 0; l < C; l++) { st.acc[l] ^= L[l]; st.Pa[l] ^= L[l]; }
    st.prev = k;
  } else if (k == a.N) {
#pragma unroll
    for (int l = 0; l < C; l++) st.Pa[l] ^= L[l];
  } else {
#pragma unroll
    for (int l = 0; l < C; l++) st.Qa[l] = L[l];
  }
}

// Epilogue: Q_xy = g^{prev} acc; class solve (Sec. 4.3 / Lemma 23.2).
__device__ __forceinline__ void finish(State& st, const ZpArgs& a, const Desc& d, const uint8_t* gexp,
                                       const uint8_t* glog, uint32_t (&o0)[C], uint32_t (&o1)[C], int& k0, int& k1) {
  mul2_n<C>(st.acc, st.prev);  // acc = Q_xy = sum_{k survivors} g^k D_k
  if (d.cls == 0) {
#pragma unroll
    for (int l = 0; l < C; l++) { o0[l] = st.Pa[l]; o1[l] = st.acc[l]; }
    k0 = a.N; k1 = a.N + 1;
  } else if (d.cls == 1) {  // D_j = P + sum D_k; Q = Q_xy + g^j D_j
    uint32_t t[C];
    mulc(st.Pa, gexp[d.x], t);
#pragma unroll
    for (int l = 0; l < C; l++) { o0[l] = st.Pa[l]; o1[l] = st.acc[l] ^ t[l]; }
    k0 = d.x; k1 = a.N + 1;
  } else if (d.cls == 2) {  // D_j = g^{-j}(Q + Q_xy); P = sum D_k
    uint32_t dq[C];
#pragma unroll
    for (int l = 0; l < C; l++) dq[l] = st.Qa[l] ^ st.acc[l];
    mulc(dq, gexp[(255 - d.x) % 255], o0);
#pragma unroll
    for (int l = 0; l < C; l++) o1[l] = st.Pa[l] ^ o0[l];
    k0 = d.x; k1 = a.N;
  } else {  // D_y = A dP + B dQ, D_x = D_y + dP
    const uint32_t A = gexp[(255 - glog[1u ^ gexp[d.y - d.x]]) % 255];
    const uint32_t B = gexp[(255 - d.x + glog[A]) % 255];
    uint32_t dq[C], t[C];
#pragma unroll
    for (int l = 0; l < C; l++) dq[l] = st.Qa[l] ^ st.acc[l];
    mulc(st.Pa, A, o1);
    mulc(dq, B, t);
#pragma unroll
    for (int l = 0; l < C; l++) { o1[l] ^= t[l]; o0[l] = o1[l] ^ st.Pa[l]; }
    k0 = d.x; k1 = d.y;
  }
}

template <bool RECOVER>
__global__ void __launch_bounds__(THREADS + 32, Cfg<RECOVER>::MINB) rs_kernel(const __grid_constant__ ZpArgs a) {
  constexpr int STAGES = Cfg<RECOVER>::STAGES;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint8_t* outb = smem + (size_t)STAGES * TB;
  uint8_t* gexp = outb + 2 * TB;  // g^k, k = 0..254
  uint8_t* glog = gexp + 256;     // log_g(v), v = 1..255
  uint64_t* full = reinterpret_cast<uint64_t*>(glog + 256);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    uint32_t v = 1;
    for (int k = 0; k < 255; k++) {
      gexp[k] = static_cast<uint8_t>(v);
      glog[v] = static_cast<uint8_t>(k);
      v = ((v << 1) & 0xffu) ^ ((v & 0x80u) ? 0x1du : 0u);
    }
    gexp[255] = 1;
    glog[0] = 0;
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], THREADS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t tiles = a.body_tiles;
  const uint64_t body_items = tiles * static_cast<uint64_t>(a.num_stripes);
  const int R = a.N;  // every class reads exactly N strips

  if (warp == THREADS / 32) {
    if (lane == 0) {
      uint32_t stage = 0, ph = 0;
      for (uint64_t it = blockIdx.x; it < body_items; it += gridDim.x) {
        const int s = static_cast<int>(it / tiles);
        const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
        const Desc d = desc_of<RECOVER>(a, s);
        for (int r = 0; r < R; r++) {
          mbar_wait(&empty[stage], ph ^ 1u);
          mbar_expect_tx(&full[stage], TB);
          tma_load_row(stages + (size_t)stage * TB, rptr(a, row_strip(a, r, d), s) + t * TB, TB, &full[stage]);
          if (++stage == STAGES) { stage = 0; ph ^= 1u; }
        }
      }
    }
    return;
  }

  uint32_t stage = 0, ph = 0;
  for (uint64_t it = blockIdx.x; it < body_items; it += gridDim.x) {
    const int s = static_cast<int>(it / tiles);
    const uint64_t t = it - static_cast<uint64_t>(s) * tiles;
    const Desc d = desc_of<RECOVER>(a, s);
    State st;
    state_init(st, a.N);
    for (int r = 0; r < R; r++) {
      const int k = row_strip(a, r, d);
      uint32_t L[C];
      mbar_wait(&full[stage], ph);
      ld_chunk_smem<C>(stages + (size_t)stage * TB + tid * CB, L);
      fold(st, a, k, L);
      consumer_release(smem_u32(&empty[stage]), lane);  // (proxy fence: see zp_fast.cuh)
      if (++stage == STAGES) { stage = 0; ph ^= 1u; }
    }
    uint32_t o0[C], o1[C];
    int k0, k1;
    finish(st, a, d, gexp, glog, o0, o1, k0, k1);
    if (tid == 0) bulk_wait_read0();
    named_bar_sync(1, THREADS);
    st_chunk_smem<C>(outb + tid * CB, o0);
    st_chunk_smem<C>(outb + TB + tid * CB, o1);
    fence_proxy_async_smem();
    named_bar_sync(1, THREADS);
    if (tid == 0) {
      tma_store_row(const_cast<uint8_t*>(rptr(a, k0, s)) + t * TB, outb, TB);
      tma_store_row(const_cast<uint8_t*>(rptr(a, k1, s)) + t * TB, outb + TB, TB);
      bulk_commit();
    }
  }

  // ragged end / unaligned strips: direct byte-precise path
  const uint64_t tups = a.tail_units_per_stripe;
  const uint64_t tail_total = tups * static_cast<uint64_t>(a.num_stripes);
  const uint64_t body_end = tiles * TB;
  for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * THREADS + tid; u < tail_total;
       u += static_cast<uint64_t>(gridDim.x) * THREADS) {
    const int s = static_cast<int>(u / tups);
    const uint64_t off = body_end + (u - static_cast<uint64_t>(s) * tups) * CB;
    const Desc d = desc_of<RECOVER>(a, s);
    State st;
    state_init(st, a.N);
#pragma unroll 1
    for (int r = 0; r < R; r++) {
      const int k = row_strip(a, r, d);
      uint32_t L[C];
      ld_chunk_global<C>(rptr(a, k, s) + off, off, a.bytes, L);
      fold(st, a, k, L);
    }
    uint32_t o0[C], o1[C];
    int k0, k1;
    finish(st, a, d, gexp, glog, o0, o1, k0, k1);
    st_chunk_global<C>(const_cast<uint8_t*>(rptr(a, k0, s)) + off, off, a.bytes, o0);
    st_chunk_global<C>(const_cast<uint8_t*>(rptr(a, k1, s)) + off, off, a.bytes, o1);
  }
  if (tid == 0) bulk_wait0();
}

}  // namespace rs

const void* rs_kernel_ptr(bool recover) {
  return recover ? reinterpret_cast<const void*>(&rs::rs_kernel<true>) : reinterpret_cast<const void*>(&rs::rs_kernel<false>);
}
size_t rs_smem_bytes(bool recover) { return recover ? rs::Cfg<true>::SMEM : rs::Cfg<false>::SMEM; }
int rs_tile_bytes() { return rs::TB; }
int rs_chunk_bytes() { return rs::CB; }
int rs_threads() { return rs::THREADS; }

}  // namespace zp
