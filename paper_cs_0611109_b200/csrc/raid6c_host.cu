// raid6c_host.cu -- host side of libraid6c: argument validation, plans, kernel selection and
// launch, and the core C ABI entry points of include/raid6c.h (the host-buffer pipeline, NEXT-3
// and NEXT-4 entry points live in host_pipeline.cu, rs_host.cu and xgpu_host.cu).
// Every byte of the method is computed by the sm_100a kernels (zp_fast.cuh / zp_generic.cu);
// there is no CPU fallback anywhere in this file.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>

#include "host_internal.h"

namespace zp {
// fast-path instantiations (zp_fast_p*.cu)
const FastEntry* fast_entry_3();
const FastEntry* fast_entry_5();
const FastEntry* fast_entry_7();
const FastEntry* fast_entry_11();
const FastEntry* fast_entry_19();
const FastEntry* fast_entry_29();
const FastEntry* fast_entry_37();
const FastEntry* fast_entry_53();
const FastEntry* fast_entry_13();
const FastEntry* fast_entry_17();
const FastEntry* fast_entry_59();
const FastEntry* fast_entry_61();
const FastEntry* fast_entry_23();
const FastEntry* fast_entry_31();
const FastEntry* fast_entry_41();
const FastEntry* fast_entry_43();
const FastEntry* fast_entry_47();
const FastEntry* fast_entry_73();
const FastEntry* fast_entry_89();
const FastEntry* fast_entry_97();
const FastEntry* fast_entry_101();
const FastEntry* fast_entry_109();
const FastEntry* fast_entry_113();
const FastEntry* fast_entry_137();
const FastEntry* fast_entry_193();
const FastEntry* fast_entry_233();
const FastEntry* fast_entry_241();
const FastEntry* fast_entry_257();

const FastEntry* fast_entry(int p) {
#ifdef ZP_SLIM  // A/B variant libraries (tools/build_variant.py --slim): the configs' primes only
  switch (p) {
    case 5: return fast_entry_5();
    case 13: return fast_entry_13();
    case 59: return fast_entry_59();
    case 61: return fast_entry_61();
    case 257: return fast_entry_257();
    default: return nullptr;
  }
#endif
  switch (p) {
    case 3: return fast_entry_3();
    case 5: return fast_entry_5();
    case 7: return fast_entry_7();
    case 11: return fast_entry_11();
    case 19: return fast_entry_19();
    case 29: return fast_entry_29();
    case 37: return fast_entry_37();
    case 53: return fast_entry_53();
    case 13: return fast_entry_13();
    case 17: return fast_entry_17();
    case 59: return fast_entry_59();
    case 61: return fast_entry_61();
    case 23: return fast_entry_23();
    case 31: return fast_entry_31();
    case 41: return fast_entry_41();
    case 43: return fast_entry_43();
    case 47: return fast_entry_47();
    case 73: return fast_entry_73();
    case 89: return fast_entry_89();
    case 97: return fast_entry_97();
    case 101: return fast_entry_101();
    case 109: return fast_entry_109();
    case 113: return fast_entry_113();
    case 137: return fast_entry_137();
    case 193: return fast_entry_193();
    case 233: return fast_entry_233();
    case 241: return fast_entry_241();
    case 257: return fast_entry_257();
    default: return nullptr;
  }
}

}  // namespace zp

namespace zp {
namespace host {

std::atomic<uint64_t> g_launches{0};
thread_local std::string g_last_err;

raid6c_status cuda_fail(cudaError_t e) {
  g_last_err = cudaGetErrorString(e);
  return RAID6C_E_CUDA;
}

bool is_valid_p(int p) {
  if (p < 3 || p > RAID6C_MAX_P || (p % 2) == 0) return false;
  for (int d = 3; d * d <= p; d += 2)
    if (p % d == 0) return false;
  return true;
}

size_t word_count(int p, size_t bytes) { return (8 * bytes + (p - 2)) / (p - 1); }
size_t parity_bytes(int p, size_t bytes) { return (word_count(p, bytes) * (p - 1) + 7) / 8; }

// ------------------------------------------------ F2[X] polynomials (64-bit limbs), host only
struct Poly {
  static constexpr int L = 10;  // 640 bits: products of two degree-<=257 polynomials fit
  uint64_t w[L] = {};
  int deg() const {
    for (int i = L - 1; i >= 0; i--)
      if (w[i]) return 64 * i + 63 - __builtin_clzll(w[i]);
    return -1;
  }
  bool bit(int i) const { return (w[i >> 6] >> (i & 63)) & 1u; }
  void flip(int i) { w[i >> 6] ^= 1ull << (i & 63); }
  void xor_shifted(const Poly& b, int sh) {  // this ^= b * X^sh
    const int q = sh >> 6, r = sh & 63;
    for (int i = L - 1; i >= q; i--) {
      uint64_t v = b.w[i - q] << r;
      if (r && i - q - 1 >= 0) v |= b.w[i - q - 1] >> (64 - r);
      w[i] ^= v;
    }
  }
  bool is_one() const {
    if (w[0] != 1) return false;
    for (int i = 1; i < L; i++)
      if (w[i]) return false;
    return true;
  }
  bool is_zero() const { return deg() < 0; }
};

Poly pmul(const Poly& a, const Poly& b) {
  Poly r;
  for (int i = 0, d = a.deg(); i <= d; i++)
    if (a.bit(i)) r.xor_shifted(b, i);
  return r;
}
void pdivmod(Poly a, const Poly& b, Poly& q, Poly& r) {  // a = q b + r
  q = Poly();
  const int db = b.deg();
  for (int da = a.deg(); da >= db; da = a.deg()) {
    q.flip(da - db);
    a.xor_shifted(b, da - db);
  }
  r = a;
}
Poly pgcd(Poly a, Poly b) {
  while (!b.is_zero()) {
    Poly q, r;
    pdivmod(a, b, q, r);
    a = b;
    b = r;
  }
  return a;
}

// Theorem 25.3 condition (3): gcd(X^p + 1, X^m + X + 1) = 1 for 0 < m < p.
bool ext_supported_p(int p) {
  Poly xp1;
  xp1.flip(p);
  xp1.flip(0);
  for (int m = 1; m < p; m++) {
    Poly t;
    t.flip(m);
    t.flip(1);
    t.flip(0);
    if (!pgcd(xp1, t).is_one()) return false;
  }
  return true;
}

// Ring R_p = F2[X]/(Phi_p), Phi_p = 1 + X + ... + X^{p-1}.
Poly phi(int p) {
  Poly f;
  for (int i = 0; i < p; i++) f.flip(i);
  return f;
}
Poly ring_reduce(const Poly& a, int p) {
  Poly q, r;
  pdivmod(a, phi(p), q, r);
  return r;
}
// Q-coefficient of data strip k in Eq. (qext): X^k (k < p) or 1 + X^{k-p+1}, reduced.
Poly ext_coeff(int p, int k) {
  Poly c;
  if (k < p) {
    c.flip(k);
  } else {
    c.flip(0);
    c.flip(k - p + 1);
  }
  return ring_reduce(c, p);
}
// Inverse in R_p by the extended Euclidean algorithm; false if a is not a unit.
bool ring_inverse(const Poly& a, int p, Poly& inv) {
  Poly r0 = phi(p), r1 = ring_reduce(a, p), s0, s1;
  s1.flip(0);
  while (!r1.is_zero()) {
    Poly q, r;
    pdivmod(r0, r1, q, r);
    r0 = r1;
    r1 = r;
    Poly t = pmul(q, s1);
    for (int i = 0; i < Poly::L; i++) t.w[i] ^= s0.w[i];
    s0 = s1;
    s1 = t;
  }
  if (!r0.is_one()) return false;
  inv = ring_reduce(s0, p);
  return true;
}

// per-(device, kernel) one-time attribute setup
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_occ;  // -> CTAs per SM

raid6c_status kernel_occupancy(int device, const void* fn, int threads, size_t smem, int* occ) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto key = std::make_pair(device, fn);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) {
    *occ = it->second;
    return RAID6C_OK;
  }
  ZP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int o = 0;
  ZP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem));
  if (o < 1) o = 1;
  g_occ[key] = o;
  *occ = o;
  return RAID6C_OK;
}


raid6c_status build_prog_table(raid6c_plan pl);

raid6c_status plan_init(raid6c_plan pl, int p, int N, size_t bytes, int device, cudaStream_t stream) {
  if (!is_valid_p(p)) return RAID6C_E_INVALID_P;
  if (N < 1 || N > 2 * p - 1 || (N > p && !ext_supported_p(p))) return RAID6C_E_INVALID_N;
  if (bytes == 0) return RAID6C_E_SIZE;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0 || device < 0 || device >= ndev) {
    cudaGetLastError();
    g_last_err = "no CUDA device";
    return RAID6C_E_NO_DEVICE;
  }
  cudaDeviceProp prop;
  ZP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    g_last_err = "libraid6c is built for sm_100a only";
    return RAID6C_E_NO_DEVICE;
  }
  pl->p = p;
  pl->N = N;
  pl->bytes = bytes;
  pl->pbytes = parity_bytes(p, bytes);
  pl->device = device;
  pl->stream = stream;
  pl->num_sms = prop.multiProcessorCount;
  pl->ext = N > p;
  if (pl->ext) {
    raid6c_status st = build_prog_table(pl);
    if (st != RAID6C_OK) return st;
  }
  pl->fe = zp::fast_entry(p);
  if (pl->fe && pl->ext && !pl->fe->kernel_ext[0]) pl->fe = nullptr;  // no fast extended kernels: generic
  if (pl->fe) {
    DeviceGuard g(device);
    for (int m = 0; m < zp::NUM_KMODES; m++) {
      const void* k = pl->ext ? pl->fe->kernel_ext[m] : pl->fe->kernel[m];
      if (!k) continue;  // (no extended light-recovery kernel)
      const size_t sm = pl->ext ? pl->fe->smem_ext[m] : pl->fe->smem_bytes[m];
      raid6c_status st = kernel_occupancy(device, k, pl->fe->threads[m] + 32, sm, &pl->occ[m]);
      if (st != RAID6C_OK) return st;
    }
  }
  return RAID6C_OK;
}

void plan_release(raid6c_plan pl) {
  DeviceGuard g(pl->device);
  if (pl->d_er) cudaFree(pl->d_er);
  if (pl->d_prog) cudaFree(pl->d_prog);
  if (pl->tables_done) cudaEventDestroy(pl->tables_done);
  if (pl->d_stage) cudaFree(pl->d_stage);
  for (int i = 0; i < 3; i++)
    if (pl->hs[i]) cudaStreamDestroy(pl->hs[i]);
  for (int i = 0; i < 2; i++) {
    if (pl->ev_in[i]) cudaEventDestroy(pl->ev_in[i]);
    if (pl->ev_k[i]) cudaEventDestroy(pl->ev_k[i]);
    if (pl->ev_out[i]) cudaEventDestroy(pl->ev_out[i]);
  }
}

// Launch one batch (all stripes share p, N, bytes).  a.base / strides / erasures are set.
// mode: zp::KMODE_ENCODE / RECOVER / SCRUB / UPDATE.
raid6c_status tables_after_read(raid6c_plan pl, const zp::ZpArgs& a, cudaStream_t st);

raid6c_status launch(raid6c_plan pl, zp::ZpArgs& a, int mode, cudaStream_t st) {
  if (a.num_stripes == 0) return RAID6C_OK;
  a.N = pl->N;
  a.bytes = pl->bytes;
  a.pbytes = pl->pbytes;
  cudaError_t err;
  if (pl->fe) {
    const zp::FastEntry* fe = pl->fe;
    bool aligned = true;
    for (int k = 0; k < pl->N + 2; k++) aligned &= (reinterpret_cast<uintptr_t>(a.base[k]) & 15u) == 0;
    if (a.num_stripes > 1) aligned &= (a.data_stride % 16 == 0) && (a.parity_stride % 16 == 0);
    if (mode == zp::KMODE_UPDATE) {
      aligned &= (reinterpret_cast<uintptr_t>(a.nbase) & 15u) == 0;
      if (a.num_stripes > 1) aligned &= a.new_stride % 16 == 0;
    }
    if (mode == zp::KMODE_PARTIAL) {  // TMA stores into the owners' slots
      for (int g = 0; g < a.nranges; g++)
        aligned &= ((reinterpret_cast<uintptr_t>(a.part_p[g]) | reinterpret_cast<uintptr_t>(a.part_q[g])) & 15u) == 0;
      if (a.num_stripes > 1) aligned &= a.part_stride % 16 == 0;
    }
    const uint64_t TB = static_cast<uint64_t>(fe->tile_bytes[mode]), CB = static_cast<uint64_t>(fe->chunk_bytes[mode]);
    const int NT = fe->threads[mode];
    if (mode == zp::KMODE_COMBINE) {
      // tiles counted from range_lo; a body tile must fit every output (data strips: `bytes`)
      for (int r = 0; r < a.nsrc; r++)
        aligned &= ((reinterpret_cast<uintptr_t>(a.src_p[r]) | reinterpret_cast<uintptr_t>(a.src_q[r])) & 15u) == 0;
      if (a.num_stripes > 1) aligned &= a.part_stride % 16 == 0;
      const uint64_t lim = std::min<uint64_t>(a.range_hi, pl->bytes);
      a.body_tiles = (aligned && lim > a.range_lo) ? (lim - a.range_lo) / TB : 0;
      a.tail_units_per_stripe = (a.range_hi - a.range_lo - a.body_tiles * TB + CB - 1) / CB;
    } else {
      a.body_tiles = aligned ? pl->bytes / TB : 0;
      const uint64_t body_end = a.body_tiles * TB;
      a.tail_units_per_stripe = (pl->pbytes - body_end + CB - 1) / CB;
      a.last_tile = 0;
      // a short strip end through one partial TMA tile (kernels that support it; every row of
      // the stripe then has the same length and the rest is a multiple of 16 bytes)
      const uint64_t rest = pl->pbytes - body_end;
      // recovery takes it only in small launches (fewer items than resident CTAs): there the
      // direct tail path is the latency (config 1 literally: 22 -> 18 us per call), while in a
      // large launch a partial item costs a whole item's solve for a sliver of the data (c1
      // batched: -4.5 %); encode always (c1 batched +1.3 %)
      const bool small = (a.body_tiles + 1) * static_cast<uint64_t>(a.num_stripes) <=
                         static_cast<uint64_t>(pl->num_sms) * pl->occ[mode];
      if (aligned && !pl->ext && fe->partial_tile[mode] && pl->pbytes == pl->bytes && rest > 0 && rest % 16 == 0 &&
          (mode == zp::KMODE_ENCODE || mode == zp::KMODE_RECOVER_L || small)) {
        a.body_tiles += 1;
        a.last_tile = static_cast<uint32_t>(rest);
        a.tail_units_per_stripe = 0;
      }
    }
    const uint64_t items = a.body_tiles * static_cast<uint64_t>(a.num_stripes);
    const uint64_t tail_ctas =
        (a.tail_units_per_stripe * static_cast<uint64_t>(a.num_stripes) + NT - 1) / NT;
    const uint64_t cap = static_cast<uint64_t>(pl->num_sms) * pl->occ[mode];
    // a small launch gets separate CTAs for the tail units (latency); a large one is persistent
    uint64_t grid = items < cap ? std::min<uint64_t>(cap, items + tail_ctas)
                                : std::min<uint64_t>(cap, std::max<uint64_t>(items, tail_ctas));
    if (grid == 0) grid = 1;
    void* args[] = {&a};
    err = cudaLaunchKernel(pl->ext ? fe->kernel_ext[mode] : fe->kernel[mode], dim3(static_cast<unsigned>(grid)),
                           dim3(NT + 32), args, pl->ext ? fe->smem_ext[mode] : fe->smem_bytes[mode], st);
  } else {
    err = zp::generic_launch(a, pl->p, mode, st, pl->num_sms);
  }
  if (err != cudaSuccess) {
    pl->sticky = RAID6C_E_CUDA;
    return cuda_fail(err);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return tables_after_read(pl, a, st);
}

// Single erasure (lost_j == RAID6C_NONE, host arguments): the pair (i, Q), or (P, Q) for i = Q.
void pair_of_single(int N, int i, int& j) {
  if (j == RAID6C_NONE) j = (i == N + 1) ? N : N + 1;
}

// A copy of a host erasure list with its single erasures completed to pairs (false: none found).
bool complete_singles(int N, const raid6c_erasure* er, int count, std::vector<raid6c_erasure>& out) {
  bool any = false;
  for (int s = 0; s < count; s++) any |= er[s].lost_j == RAID6C_NONE;
  if (!any) return false;
  out.assign(er, er + count);
  for (auto& e : out) pair_of_single(N, e.lost_i, e.lost_j);
  return true;
}

raid6c_status check_erasure(int N, int i, int j) {
  if (i == j || i < 0 || j < 0 || i >= N + 2 || j >= N + 2) return RAID6C_E_INVALID_INDEX;
  return RAID6C_OK;
}

raid6c_status strided_args(raid6c_plan pl, const uint8_t* data, size_t strip_stride, size_t stripe_stride,
                           const uint8_t* P, const uint8_t* Q, size_t parity_stride, int num_stripes,
                           zp::ZpArgs& a) {
  if (!pl) return RAID6C_E_NULL;
  if (num_stripes < 0) return RAID6C_E_SIZE;
  if (!data || !P || !Q) return RAID6C_E_NULL;
  if (pl->N > 1 && strip_stride < pl->bytes) return RAID6C_E_SIZE;
  if (num_stripes > 1 && (stripe_stride < pl->bytes || parity_stride < pl->pbytes)) return RAID6C_E_SIZE;
  std::memset(&a, 0, sizeof(a));
  for (int k = 0; k < pl->N; k++) a.base[k] = data + static_cast<size_t>(k) * strip_stride;
  a.base[pl->N] = P;
  a.base[pl->N + 1] = Q;
  a.data_stride = stripe_stride;
  a.parity_stride = parity_stride;
  a.num_stripes = num_stripes;
  a.ei = pl->N;
  a.ej = pl->N + 1;
  return RAID6C_OK;
}

// NEXT-4 combine + solve over bytes [a.range_lo, a.range_hi) of every stripe.
raid6c_status launch_combine(raid6c_plan pl, zp::ZpArgs& a, cudaStream_t st) {
  if (a.num_stripes == 0 || a.range_hi <= a.range_lo) return RAID6C_OK;
  return launch(pl, a, zp::KMODE_COMBINE, st);
}

// Word-range granule of p's kernels: a TMA tile (fast path) or lcm(byte group, 16) (generic).
uint64_t range_granule_p(int p) {
  // ranges are whole tiles of the partial kernel (a tile has one owner); the combine kernel
  // starts its own tiles at each range start (16-byte and word aligned)
  if (const zp::FastEntry* fe = zp::fast_entry(p)) return static_cast<uint64_t>(fe->tile_bytes[zp::KMODE_PARTIAL]);
  const int n = p - 1;
  const int g = 8 / (n & 7 ? ((n & 3) ? 2 : 4) : 8);
  const uint64_t gb = static_cast<uint64_t>(g) * n / 8;
  return gb * 16 / std::gcd<uint64_t>(gb, 16);
}
uint64_t range_granule(raid6c_plan pl) {
  if (pl->fe) return static_cast<uint64_t>(pl->fe->tile_bytes[zp::KMODE_PARTIAL]);
  return range_granule_p(pl->p);
}

// Order a rewrite of the plan's device tables (d_er, d_prog) on stream st after every launch
// that reads them; `freeing` = the buffer is about to be released (wait on the host instead).
raid6c_status tables_before_write(raid6c_plan pl, cudaStream_t st, bool freeing) {
#ifdef ZP_NO_TABLE_ORDER  // negative control for tests/test_gpu_parity.py (never in the product build)
  return RAID6C_OK;
#endif
  if (!pl->tables_pending) return RAID6C_OK;
  if (freeing) {
    ZP_CUDA(cudaEventSynchronize(pl->tables_done));
    pl->tables_pending = false;
    return RAID6C_OK;
  }
  ZP_CUDA(cudaStreamWaitEvent(st, pl->tables_done, 0));
  return RAID6C_OK;
}

// After a launch on st whose arguments point into d_er / d_prog.
raid6c_status tables_after_read(raid6c_plan pl, const zp::ZpArgs& a, cudaStream_t st) {
  const bool uses_er = pl->d_er && ((a.er >= pl->d_er && a.er < pl->d_er + pl->er_cap) ||
                                    (reinterpret_cast<const int2*>(a.upd) >= pl->d_er &&
                                     reinterpret_cast<const int2*>(a.upd) < pl->d_er + pl->er_cap));
  if (!uses_er) return RAID6C_OK;  // (the extended code's program table is never rewritten)
  if (!pl->tables_done) ZP_CUDA(cudaEventCreateWithFlags(&pl->tables_done, cudaEventDisableTiming));
  ZP_CUDA(cudaEventRecord(pl->tables_done, st));
  pl->tables_pending = true;
  return RAID6C_OK;
}

// Upload host erasure pairs (validated, canonical) into the plan's device buffer.
raid6c_status upload_erasures(raid6c_plan pl, const raid6c_erasure* er, int count, cudaStream_t st) {
  std::vector<int2> h(count);
  for (int s = 0; s < count; s++) {
    const int i = er[s].lost_i, j = er[s].lost_j;
    raid6c_status e = check_erasure(pl->N, i, j);
    if (e != RAID6C_OK) return e;
    h[s] = make_int2(std::min(i, j), std::max(i, j));
  }
  if (static_cast<size_t>(count) > pl->er_cap) {
    DeviceGuard g(pl->device);
    if (pl->d_er) {
      ZP_CUDA(cudaStreamSynchronize(st));
      raid6c_status w = tables_before_write(pl, st, true);
      if (w != RAID6C_OK) return w;
      cudaFree(pl->d_er);
      pl->d_er = nullptr;
    }
    size_t cap = std::max<size_t>(1024, static_cast<size_t>(count));
    ZP_CUDA(cudaMalloc(&pl->d_er, cap * sizeof(int2)));
    pl->er_cap = cap;
  }
  raid6c_status w = tables_before_write(pl, st, false);
  if (w != RAID6C_OK) return w;
  // pageable source: the copy is staged before this call returns, so `h` may be freed
  ZP_CUDA(cudaMemcpyAsync(pl->d_er, h.data(), count * sizeof(int2), cudaMemcpyHostToDevice, st));
  return RAID6C_OK;
}

// Extended code: the multiplier u of the DP / DD solve of pair (x, y), x < y (ExtProg).
raid6c_status make_prog(int p, int N, int x, int y, zp::ExtProg& pr) {
  std::memset(&pr, 0, sizeof(pr));
  // Geometric pairs (kernel: series of the basic code instead of the exponent list):
  //   DP, j >= p:          g_j^{-1} = (1 + x^c)^{-1},            c = j - p + 1
  //   DD, x < y < p:       (x^x + x^y)^{-1} = x^{-x} (1 + x^{y-x})^{-1}
  //   DD, p <= x < y:      (x^cx + x^cy)^{-1} = x^{-cx} (1 + x^{cy-cx})^{-1},  c = k - p + 1
  if (y == N && x >= p) {
    pr.geo_bz = static_cast<int16_t>((2 * (x - p + 1)) % p);
    return RAID6C_OK;
  }
  if (y < N && (y < p || x >= p)) {
    const int ex = x < p ? x : x - p + 1, ey = y < p ? y : y - p + 1;
    pr.geo_bz = static_cast<int16_t>((2 * (ey - ex)) % p);
    pr.geo_e0 = static_cast<int16_t>((p - ex) % p);
    return RAID6C_OK;
  }
  Poly c;
  if (y == N + 1) return RAID6C_OK;  // DQ / PQ: no solve
  if (y == N) {                      // DP, j < p: u = g_j^{-1} = x^{p-j}
    c = ext_coeff(p, x);
  } else {                           // DD, mixed pair: u = (x^a + 1 + x^c)^{-1}
    c = ext_coeff(p, x);
    Poly cy = ext_coeff(p, y);
    for (int i = 0; i < Poly::L; i++) c.w[i] ^= cy.w[i];
  }
  Poly u;
  if (!ring_inverse(c, p, u)) {
    g_last_err = "extended code: coefficient not invertible";
    return RAID6C_E_INVALID_N;
  }
  for (int i = 0; i < p - 1; i++)
    if (u.bit(i)) pr.e[pr.nu++] = static_cast<uint16_t>(i);
  // u and u + (1 + x + ... + x^{p-1}) are the same element of R_p (the p-th roots of unity
  // sum to zero, Lemma 24.2), and the kernel multiplies in R' with
  // deferred reduction: take whichever has fewer terms (the complement includes x^{p-1}).
  if (2 * pr.nu > p) {
    int k = 0;
    for (int i = 0; i < p; i++)
      if (i == p - 1 || !u.bit(i)) pr.e[k++] = static_cast<uint16_t>(i);
    pr.nu = k;
  }
  return RAID6C_OK;
}

// Extended-code plans: the multipliers of every pair, indexed by zp::pair_index, built and
// uploaded once at plan creation -- so a recovery whose per-stripe pairs live on the device
// needs no host round trip.
raid6c_status build_prog_table(raid6c_plan pl) {
  const int p = pl->p, N = pl->N, K = N + 2;
  const size_t n = static_cast<size_t>(K) * (K - 1) / 2;
  std::vector<zp::ExtProg> h(n);
  for (int x = 0; x < K; x++)
    for (int y = x + 1; y < K; y++) {
      raid6c_status st = make_prog(p, N, x, y, h[zp::pair_index(x, y, N)]);
      if (st != RAID6C_OK) return st;
    }
  DeviceGuard g(pl->device);
  ZP_CUDA(cudaMalloc(&pl->d_prog, n * sizeof(zp::ExtProg)));
  pl->prog_cap = n;
  ZP_CUDA(cudaMemcpy(pl->d_prog, h.data(), n * sizeof(zp::ExtProg), cudaMemcpyHostToDevice));
  return RAID6C_OK;
}

// Erasure pairs of a batched call into the launch args (host array: validated and uploaded or
// passed by value; device array: used in place).  with_programs: the extended code's
// per-stripe multipliers (ExtProg) for the DP / DD solves are built and uploaded too.
raid6c_status set_erasures(raid6c_plan plan, zp::ZpArgs& a, const raid6c_erasure* erasures, int num_erasures,
                           int erasures_on_device, int num_stripes, bool with_programs) {
  raid6c_status st = RAID6C_OK;
  if (num_erasures != 1 && num_erasures != num_stripes) return RAID6C_E_SIZE;
  if (plan->ext && with_programs) a.prog = plan->d_prog;  // per-pair table (build_prog_table)
  if (erasures_on_device) {
    a.er = reinterpret_cast<const int2*>(erasures);
    a.er_stride = num_erasures == 1 ? 0 : 1;
  } else if (num_erasures == 1) {
    st = check_erasure(plan->N, erasures[0].lost_i, erasures[0].lost_j);
    if (st != RAID6C_OK) return st;
    a.ei = std::min(erasures[0].lost_i, erasures[0].lost_j);
    a.ej = std::max(erasures[0].lost_i, erasures[0].lost_j);
  } else {
    for (int s = 0; s < num_erasures; s++) {
      st = check_erasure(plan->N, erasures[s].lost_i, erasures[s].lost_j);
      if (st != RAID6C_OK) return st;
    }
    st = upload_erasures(plan, erasures, num_erasures, plan->stream);
    if (st != RAID6C_OK) return st;
    a.er = plan->d_er;
    a.er_stride = 1;
  }
  return RAID6C_OK;
}

// True when every (host) erasure pair is {P, Q} = {N, N+1}, in either order.
bool pq_only(int N, const raid6c_erasure* er, int count) {
  if (count < 1) return false;
  for (int s = 0; s < count; s++) {
    const int i = std::min(er[s].lost_i, er[s].lost_j), j = std::max(er[s].lost_i, er[s].lost_j);
    if (i != N || j != N + 1) return false;
  }
  return true;
}

// True when no (host) erasure pair is class DD (every pair loses P or Q).
bool no_dd(int N, const raid6c_erasure* er, int count) {
  if (count < 1) return false;
  for (int s = 0; s < count; s++)
    if (std::max(er[s].lost_i, er[s].lost_j) < N) return false;
  return true;
}

// ------------------------------------------------------------------ cached single-stripe plans
// The north-star calls share one plan per (device, p, N, bytes).  Callers hold the plan through
// a shared_ptr for the whole call, so evicting an entry (the cache is bounded) only drops the
// cache's reference: a plan is released when its last in-flight call returns, never under it.
std::mutex g_cache_mu;
std::map<std::tuple<int, int, int, size_t>, std::shared_ptr<raid6c_plan_s>> g_cache;
constexpr size_t kCacheMax = 64;

raid6c_status cached_plan(int p, int N, size_t bytes, std::shared_ptr<raid6c_plan_s>* out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    g_last_err = "no CUDA device";
    return RAID6C_E_NO_DEVICE;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto key = std::make_tuple(dev, p, N, bytes);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    *out = it->second;
    return RAID6C_OK;
  }
  std::shared_ptr<raid6c_plan_s> pl(new raid6c_plan_s(), [](raid6c_plan_s* q) {
    plan_release(q);
    delete q;
  });
  raid6c_status st = plan_init(pl.get(), p, N, bytes, dev, nullptr);
  if (st != RAID6C_OK) return st;  // (the deleter releases what plan_init allocated)
  if (g_cache.size() >= kCacheMax) g_cache.erase(g_cache.begin());  // one entry; in-use plans live on
  g_cache[key] = pl;
  *out = std::move(pl);
  return RAID6C_OK;
}

}  // namespace host
}  // namespace zp

using namespace zp::host;

// ====================================================================== C ABI
extern "C" {

size_t raid6c_word_count(int p, size_t bytes) { return is_valid_p(p) ? word_count(p, bytes) : 0; }
size_t raid6c_parity_bytes(int p, size_t bytes) { return is_valid_p(p) ? parity_bytes(p, bytes) : 0; }
int raid6c_valid_p(int p) { return is_valid_p(p) ? 1 : 0; }
int raid6c_has_fast_path(int p) { return zp::fast_entry(p) != nullptr ? 1 : 0; }
int raid6c_ext_supported(int p) { return is_valid_p(p) && ext_supported_p(p) ? 1 : 0; }
uint64_t raid6c_launch_count(void) { return g_launches.load(); }
const char* raid6c_last_cuda_error(void) { return g_last_err.c_str(); }

const char* raid6c_status_string(raid6c_status s) {
  switch (s) {
    case RAID6C_OK: return "ok";
    case RAID6C_E_INVALID_P: return "p is not an odd prime in [3, 257]";
    case RAID6C_E_INVALID_N: return "N must satisfy 1 <= N <= p, or p < N <= 2p-1 with p satisfying Theorem 25.3";
    case RAID6C_E_INVALID_INDEX: return "lost strip index out of range or repeated";
    case RAID6C_E_NULL: return "null pointer argument";
    case RAID6C_E_SIZE: return "invalid size or stride";
    case RAID6C_E_CUDA: return "CUDA error";
    case RAID6C_E_NO_DEVICE: return "no usable sm_100 CUDA device";
    case RAID6C_E_PLAN: return "call does not match the plan";
  }
  return "unknown status";
}

raid6c_status raid6c_plan_create(raid6c_plan* out, int p, int N, size_t bytes, int device, void* stream) {
  if (!out) return RAID6C_E_NULL;
  *out = nullptr;
  raid6c_plan pl = new raid6c_plan_s();
  raid6c_status st = plan_init(pl, p, N, bytes, device, static_cast<cudaStream_t>(stream));
  if (st != RAID6C_OK) {
    plan_release(pl);  // (buffers allocated before the failure, e.g. the program table)
    delete pl;
    return st;
  }
  *out = pl;
  return RAID6C_OK;
}

raid6c_status raid6c_plan_destroy(raid6c_plan plan) {
  if (!plan) return RAID6C_E_NULL;
  {
    DeviceGuard g(plan->device);
    cudaStreamSynchronize(plan->stream);
    for (int i = 0; i < 3; i++)
      if (plan->hs[i]) cudaStreamSynchronize(plan->hs[i]);
  }
  plan_release(plan);
  delete plan;
  return RAID6C_OK;
}

raid6c_status raid6c_plan_set_stream(raid6c_plan plan, void* stream) {
  if (!plan) return RAID6C_E_NULL;
  plan->stream = static_cast<cudaStream_t>(stream);
  return RAID6C_OK;
}

raid6c_status raid6c_sync(raid6c_plan plan) {
  if (!plan) return RAID6C_E_NULL;
  DeviceGuard g(plan->device);
  cudaError_t e = cudaStreamSynchronize(plan->stream);
  raid6c_status st = plan->sticky;
  plan->sticky = RAID6C_OK;
  if (e != cudaSuccess) return cuda_fail(e);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  return st;
}

raid6c_status raid6c_encode(int p, int N, const uint8_t* const* strips, uint8_t* P, uint8_t* Q, size_t bytes) {
  if (!is_valid_p(p)) return RAID6C_E_INVALID_P;
  if (N < 1 || N > 2 * p - 1 || (N > p && !ext_supported_p(p))) return RAID6C_E_INVALID_N;
  if (bytes == 0) return RAID6C_E_SIZE;
  if (!strips || !P || !Q) return RAID6C_E_NULL;
  for (int k = 0; k < N; k++)
    if (!strips[k]) return RAID6C_E_NULL;
  std::shared_ptr<raid6c_plan_s> hold;
  raid6c_status st = cached_plan(p, N, bytes, &hold);
  if (st != RAID6C_OK) return st;
  raid6c_plan pl = hold.get();
  zp::ZpArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int k = 0; k < N; k++) a.base[k] = strips[k];
  a.base[N] = P;
  a.base[N + 1] = Q;
  a.num_stripes = 1;
  a.ei = N;
  a.ej = N + 1;
  st = launch(pl, a, zp::KMODE_ENCODE, nullptr);
  if (st != RAID6C_OK) return st;
  ZP_CUDA(cudaStreamSynchronize(nullptr));
  ZP_CUDA(cudaGetLastError());
  return RAID6C_OK;
}

raid6c_status raid6c_recover(int p, int N, int lost_i, int lost_j, uint8_t* const* strips, size_t bytes) {
  if (!is_valid_p(p)) return RAID6C_E_INVALID_P;
  if (N < 1 || N > 2 * p - 1 || (N > p && !ext_supported_p(p))) return RAID6C_E_INVALID_N;
  if (bytes == 0) return RAID6C_E_SIZE;
  pair_of_single(N, lost_i, lost_j);
  raid6c_status st = check_erasure(N, lost_i, lost_j);
  if (st != RAID6C_OK) return st;
  if (!strips) return RAID6C_E_NULL;
  for (int k = 0; k < N + 2; k++)
    if (!strips[k]) return RAID6C_E_NULL;
  std::shared_ptr<raid6c_plan_s> hold;
  st = cached_plan(p, N, bytes, &hold);
  if (st != RAID6C_OK) return st;
  raid6c_plan pl = hold.get();
  zp::ZpArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int k = 0; k < N + 2; k++) a.base[k] = strips[k];
  a.num_stripes = 1;
  a.ei = std::min(lost_i, lost_j);
  a.ej = std::max(lost_i, lost_j);
  std::unique_lock<std::mutex> lk(pl->mu);
  const bool pq = a.ei == N && a.ej == N + 1;  // class PQ: the rebuild is the encode
  if (pl->ext && !pq) a.prog = pl->d_prog;
  const bool light = !pq && pl->fe && !pl->ext && a.ej >= N;  // DP / DQ: light recovery kernel
  st = launch(pl, a, pq ? zp::KMODE_ENCODE : (light ? zp::KMODE_RECOVER_L : zp::KMODE_RECOVER), nullptr);
  if (st != RAID6C_OK) return st;
  ZP_CUDA(cudaStreamSynchronize(nullptr));
  ZP_CUDA(cudaGetLastError());
  return RAID6C_OK;
}

raid6c_status raid6c_encode_strided(raid6c_plan plan, const uint8_t* data, size_t strip_stride, size_t stripe_stride,
                                    uint8_t* P, uint8_t* Q, size_t parity_stride, int num_stripes) {
  zp::ZpArgs a;
  raid6c_status st = strided_args(plan, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, a);
  if (st != RAID6C_OK) return st;
  DeviceGuard g(plan->device);
  return launch(plan, a, zp::KMODE_ENCODE, plan->stream);
}

raid6c_status raid6c_recover_strided(raid6c_plan plan, uint8_t* data, size_t strip_stride, size_t stripe_stride,
                                     uint8_t* P, uint8_t* Q, size_t parity_stride, int num_stripes,
                                     const raid6c_erasure* erasures, int num_erasures, int erasures_on_device) {
  zp::ZpArgs a;
  raid6c_status st = strided_args(plan, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, a);
  if (st != RAID6C_OK) return st;
  if (!erasures) return RAID6C_E_NULL;
  std::vector<raid6c_erasure> completed;  // single erasures (RAID6C_NONE) as pairs
  if (!erasures_on_device && num_erasures >= 1 && complete_singles(plan->N, erasures, num_erasures, completed))
    erasures = completed.data();
  DeviceGuard g(plan->device);
  // Both parity strips lost in every stripe (class PQ, known on the host): the rebuild IS the
  // encode (Eq. (znparity)), so it runs on the encode kernel (lighter geometry, 3 CTAs/SM where
  // that wins) instead of the recovery kernel's PQ branch.
  if (!erasures_on_device && pq_only(plan->N, erasures, num_erasures)) {
    a.ei = plan->N;
    a.ej = plan->N + 1;
    return launch(plan, a, zp::KMODE_ENCODE, plan->stream);
  }
  st = set_erasures(plan, a, erasures, num_erasures, erasures_on_device, num_stripes, true);
  if (st != RAID6C_OK) return st;
  // No DD stripe in the launch (known on the host): the light recovery kernel (encode geometry;
  // fast path, basic code)
  const bool light = !erasures_on_device && plan->fe && !plan->ext && no_dd(plan->N, erasures, num_erasures);
  return launch(plan, a, light ? zp::KMODE_RECOVER_L : zp::KMODE_RECOVER, plan->stream);
}

raid6c_status raid6c_scrub_strided(raid6c_plan plan, const uint8_t* data, size_t strip_stride, size_t stripe_stride,
                                   const uint8_t* P, const uint8_t* Q, size_t parity_stride, int num_stripes,
                                   uint32_t* bad_words) {
  zp::ZpArgs a;
  raid6c_status st = strided_args(plan, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, a);
  if (st != RAID6C_OK) return st;
  if (!bad_words) return RAID6C_E_NULL;
  if (num_stripes == 0) return RAID6C_OK;
  DeviceGuard g(plan->device);
  ZP_CUDA(cudaMemsetAsync(bad_words, 0, static_cast<size_t>(num_stripes) * sizeof(uint32_t), plan->stream));
  a.counts = bad_words;
  return launch(plan, a, zp::KMODE_SCRUB, plan->stream);
}

raid6c_status raid6c_update_strided(raid6c_plan plan, uint8_t* data, size_t strip_stride, size_t stripe_stride,
                                    uint8_t* P, uint8_t* Q, size_t parity_stride, int num_stripes,
                                    const uint8_t* new_data, size_t new_stride, const int32_t* disks, int num_disks,
                                    int disks_on_device) {
  zp::ZpArgs a;
  raid6c_status st = strided_args(plan, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, a);
  if (st != RAID6C_OK) return st;
  if (!new_data || !disks) return RAID6C_E_NULL;
  if (num_disks != 1 && num_disks != num_stripes) return RAID6C_E_SIZE;
  if (num_stripes > 1 && new_stride < plan->bytes) return RAID6C_E_SIZE;
  a.nbase = new_data;
  a.new_stride = new_stride;
  a.upd_rows = 4;
  DeviceGuard g(plan->device);
  if (disks_on_device) {
    a.upd = disks;
    a.upd_stride = num_disks == 1 ? 0 : 1;
  } else if (num_disks == 1) {
    if (disks[0] < 0 || disks[0] >= plan->N) return RAID6C_E_INVALID_INDEX;
    a.upd_k = disks[0];
  } else {
    std::vector<raid6c_erasure> ev(num_disks);
    for (int s = 0; s < num_disks; s++) {
      if (disks[s] < 0 || disks[s] >= plan->N) return RAID6C_E_INVALID_INDEX;
      ev[s] = {disks[s], plan->N};  // packed as (k, N): the kernel reads .x only
    }
    st = upload_erasures(plan, ev.data(), num_disks, plan->stream);
    if (st != RAID6C_OK) return st;
    a.upd = reinterpret_cast<const int32_t*>(plan->d_er);
    a.upd_stride = 2;
  }
  return launch(plan, a, zp::KMODE_UPDATE, plan->stream);
}

raid6c_status raid6c_fill(uint8_t* dst, size_t strip_stride, size_t stripe_stride, size_t len, int nstrips,
                          int nstripes, uint64_t seed, int cfg, int stripe0, int strip0, int sparse_mode,
                          void* stream) {
  if (!dst) return RAID6C_E_NULL;
  if (nstrips < 0 || nstripes < 0) return RAID6C_E_SIZE;
  if (len == 0 || nstrips == 0 || nstripes == 0) return RAID6C_OK;
  cudaError_t e = zp::harness_fill(dst, strip_stride, stripe_stride, len, nstrips, nstripes, seed, cfg, stripe0, strip0,
                                   sparse_mode, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return RAID6C_OK;
}

raid6c_status raid6c_count_mismatch(const uint8_t* a, const uint8_t* b, size_t len, uint64_t* count_dev, void* stream) {
  if (!a || !b || !count_dev) return RAID6C_E_NULL;
  if (len == 0) return RAID6C_OK;
  cudaError_t e = zp::harness_count_mismatch(a, b, len, count_dev, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return RAID6C_OK;
}

raid6c_status raid6c_digest(const uint8_t* src, size_t strip_stride, size_t stripe_stride, size_t len, int nstrips,
                            int nstripes, uint64_t* digests_dev, void* stream) {
  if (!src || !digests_dev) return RAID6C_E_NULL;
  if (nstrips < 0 || nstripes < 0) return RAID6C_E_SIZE;
  if (nstrips == 0 || nstripes == 0) return RAID6C_OK;
  cudaError_t e = zp::harness_digest(src, strip_stride, stripe_stride, len, nstrips, nstripes, digests_dev,
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return RAID6C_OK;
}

}  // extern "C"
