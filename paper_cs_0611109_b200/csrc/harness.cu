// harness.cu -- bench/test harness kernels (NOT the method): the synthetic generator of
// synthetic/gen.py re-implemented on the device (checked bit-for-bit against the numpy
// version by tests/test_gpu_parity.py::test_fill_matches_numpy_generator), a byte compare, and
// a per-strip 64-bit digest (synthetic/digest.py; tests/test_gpu_digest.py) that lets full-size
// GPU outputs be compared with oracle outputs computed elsewhere (host cores, other ranks).
#include <cstdint>
#include <cuda_runtime.h>

namespace zp {
namespace {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t SPARSE_A = 0xA5A5A5A55A5A5A5Aull;
constexpr uint64_t SPARSE_B = 0x3C3C3C3CC3C3C3C3ull;
constexpr uint32_t SPARSE_ZERO_BELOW = 58982u;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__global__ void fill_kernel(uint8_t* dst, uint64_t strip_stride, uint64_t stripe_stride, uint64_t len, int nstrips,
                            int nstripes, uint64_t seed, int cfg, int stripe0, int strip0, int sparse_mode) {
  const uint64_t wps = (len + 7) / 8;
  const uint64_t total = wps * static_cast<uint64_t>(nstrips) * static_cast<uint64_t>(nstripes);
  for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < total;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = u % wps;
    const uint64_t st = u / wps;
    const int t = static_cast<int>(st % nstrips);
    const int s = static_cast<int>(st / nstrips);
    const uint64_t gs = static_cast<uint64_t>(stripe0 + s), gt = static_cast<uint64_t>(strip0 + t);
    const uint64_t hi = ((((static_cast<uint64_t>(cfg) * 8192u + gs) * 512u + gt) << 22) + seed * GOLDEN);
    const uint64_t key = hi + k;
    uint64_t v = mix64(key);
    const bool sparse = sparse_mode == 1 || (sparse_mode == 2 && (gs & 1u));
    if (sparse) {
      const uint64_t da = mix64(key ^ SPARSE_A), db = mix64(key ^ SPARSE_B);
      uint64_t out = 0;
#pragma unroll
      for (int b = 0; b < 8; b++) {
        const uint32_t draw = static_cast<uint32_t>(((b < 4 ? da : db) >> (16 * (b & 3))) & 0xFFFFu);
        const uint32_t byte = static_cast<uint32_t>((v >> (8 * b)) & 0xFFu);
        const uint32_t nz = 1u + byte % 255u;
        out |= static_cast<uint64_t>(draw < SPARSE_ZERO_BELOW ? 0u : nz) << (8 * b);
      }
      v = out;
    }
    uint8_t* p = dst + static_cast<uint64_t>(s) * stripe_stride + static_cast<uint64_t>(t) * strip_stride + 8 * k;
    if (8 * k + 8 <= len && (reinterpret_cast<uintptr_t>(p) & 7u) == 0) {
      *reinterpret_cast<uint64_t*>(p) = v;
    } else {
      for (int b = 0; b < 8; b++)
        if (8 * k + b < len) p[b] = static_cast<uint8_t>(v >> (8 * b));
    }
  }
}

__global__ void count_mismatch_kernel(const uint8_t* a, const uint8_t* b, uint64_t len, unsigned long long* out) {
  unsigned long long c = 0;
  const bool al = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15u) == 0;
  const uint64_t nv = al ? len / 16 : 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint4 x = reinterpret_cast<const uint4*>(a)[i], y = reinterpret_cast<const uint4*>(b)[i];
    const uint32_t d[4] = {x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w};
    for (int j = 0; j < 4; j++)
      for (int q = 0; q < 4; q++) c += ((d[j] >> (8 * q)) & 0xFFu) != 0;
  }
  for (uint64_t i = nv * 16 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    c += a[i] != b[i];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Per-strip digest (harness, not the method; synthetic/digest.py is the host version):
//   digest(b) = mix64(len ^ DIGEST_LEN) + sum_k mix64(w_k + k * GOLDEN + DIGEST_DOMAIN)  (mod 2^64)
// w_k = little-endian u64 of bytes [8k, 8k+8), zero past len.  mix64 is a bijection, so one
// changed word always changes its term; the sum is order-free, so blocks add their part with
// one wrapping 64-bit atomic per warp.
constexpr uint64_t DIGEST_DOMAIN = 0x6A09E667F3BCC909ull;
constexpr uint64_t DIGEST_LEN = 0xBB67AE8584CAA73Bull;
constexpr int DIGEST_SEG_WORDS = 4096;  // words per block work unit (32 KiB)

__global__ void digest_init_kernel(unsigned long long* out, uint64_t n, uint64_t len) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = mix64(len ^ DIGEST_LEN);
}

__global__ void digest_kernel(const uint8_t* src, uint64_t strip_stride, uint64_t stripe_stride, uint64_t len,
                              int nstrips, int nstripes, unsigned long long* out) {
  const uint64_t wps = (len + 7) / 8;
  const uint64_t segs = (wps + DIGEST_SEG_WORDS - 1) / DIGEST_SEG_WORDS;
  const uint64_t units = segs * static_cast<uint64_t>(nstrips) * static_cast<uint64_t>(nstripes);
  for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const uint64_t strip = u / segs;  // = s * nstrips + t
    const uint64_t seg = u - strip * segs;
    const uint64_t s = strip / static_cast<uint64_t>(nstrips), t = strip - s * static_cast<uint64_t>(nstrips);
    const uint8_t* base = src + s * stripe_stride + t * strip_stride;
    const bool al8 = (reinterpret_cast<uintptr_t>(base) & 7u) == 0;
    const uint64_t k0 = seg * DIGEST_SEG_WORDS;
    const uint64_t k1 = k0 + DIGEST_SEG_WORDS < wps ? k0 + DIGEST_SEG_WORDS : wps;
    unsigned long long h = 0;
    for (uint64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      uint64_t w = 0;
      if (al8 && 8 * k + 8 <= len) {
        w = __ldg(reinterpret_cast<const unsigned long long*>(base) + k);
      } else {
        for (int b = 0; b < 8; b++)
          if (8 * k + b < len) w |= static_cast<uint64_t>(__ldg(base + 8 * k + b)) << (8 * b);
      }
      h += mix64(w + k * GOLDEN + DIGEST_DOMAIN);
    }
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out + strip, h);
  }
}

}  // namespace

cudaError_t harness_digest(const uint8_t* src, uint64_t strip_stride, uint64_t stripe_stride, uint64_t len,
                           int nstrips, int nstripes, uint64_t* out, cudaStream_t st) {
  const uint64_t n = static_cast<uint64_t>(nstrips) * static_cast<uint64_t>(nstripes);
  auto* o = reinterpret_cast<unsigned long long*>(out);
  uint64_t ib = (n + 255) / 256;
  digest_init_kernel<<<static_cast<unsigned>(ib < 1024 ? (ib ? ib : 1) : 1024), 256, 0, st>>>(o, n, len);
  const uint64_t units = ((len + 7) / 8 + DIGEST_SEG_WORDS - 1) / DIGEST_SEG_WORDS * n;
  uint64_t blocks = units < 148ull * 8 ? units : 148ull * 8;
  if (blocks == 0) blocks = 1;
  digest_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(src, strip_stride, stripe_stride, len, nstrips,
                                                               nstripes, o);
  return cudaGetLastError();
}

cudaError_t harness_fill(uint8_t* dst, uint64_t strip_stride, uint64_t stripe_stride, uint64_t len, int nstrips,
                         int nstripes, uint64_t seed, int cfg, int stripe0, int strip0, int sparse_mode,
                         cudaStream_t st) {
  const uint64_t total = ((len + 7) / 8) * static_cast<uint64_t>(nstrips) * static_cast<uint64_t>(nstripes);
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  if (blocks == 0) blocks = 1;
  fill_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(dst, strip_stride, stripe_stride, len, nstrips, nstripes,
                                                             seed, cfg, stripe0, strip0, sparse_mode);
  return cudaGetLastError();
}

cudaError_t harness_count_mismatch(const uint8_t* a, const uint8_t* b, uint64_t len, uint64_t* out, cudaStream_t st) {
  uint64_t blocks = (len / 16 + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (blocks == 0) blocks = 1;
  count_mismatch_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(a, b, len,
                                                                       reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

}  // namespace zp
