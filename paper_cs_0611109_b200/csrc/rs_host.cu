// rs_host.cu -- NEXT-3 entry points of libraid6c: the paper's GF(256) Reed-Solomon comparison
// system (rs.cu kernels) launched on the same pipeline and conventions as the Z_p calls.
#include <algorithm>
#include <cstring>
#include <vector>

#include "host_internal.h"

using namespace zp::host;

extern "C" {

// ---------------------------------------------------------------- NEXT-3: GF(256) RS baseline
static raid6c_status rs_launch(int N, size_t bytes, const uint8_t* data, size_t strip_stride, size_t stripe_stride,
                               const uint8_t* P, const uint8_t* Q, size_t parity_stride, int num_stripes, bool recover,
                               const raid6c_erasure* er, int num_er, int er_on_device, cudaStream_t st) {
  if (N < 1 || N > 255) return RAID6C_E_INVALID_N;
  if (bytes == 0 || num_stripes < 0) return RAID6C_E_SIZE;
  if (!data || !P || !Q) return RAID6C_E_NULL;
  if (N > 1 && strip_stride < bytes) return RAID6C_E_SIZE;
  if (num_stripes > 1 && (stripe_stride < bytes || parity_stride < bytes)) return RAID6C_E_SIZE;
  if (num_stripes == 0) return RAID6C_OK;
  zp::ZpArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int k = 0; k < N; k++) a.base[k] = data + static_cast<size_t>(k) * strip_stride;
  a.base[N] = P;
  a.base[N + 1] = Q;
  a.data_stride = stripe_stride;
  a.parity_stride = parity_stride;
  a.bytes = a.pbytes = bytes;
  a.N = N;
  a.num_stripes = num_stripes;
  a.ei = N;
  a.ej = N + 1;
  int2* tmp = nullptr;
  if (recover) {
    if (!er) return RAID6C_E_NULL;
    if (num_er != 1 && num_er != num_stripes) return RAID6C_E_SIZE;
    if (er_on_device) {
      a.er = reinterpret_cast<const int2*>(er);
      a.er_stride = num_er == 1 ? 0 : 1;
    } else {
      std::vector<int2> h(num_er);
      for (int s = 0; s < num_er; s++) {
        raid6c_status c = check_erasure(N, er[s].lost_i, er[s].lost_j);
        if (c != RAID6C_OK) return c;
        h[s] = make_int2(std::min(er[s].lost_i, er[s].lost_j), std::max(er[s].lost_i, er[s].lost_j));
      }
      if (num_er == 1) {
        a.ei = h[0].x;
        a.ej = h[0].y;
      } else {
        ZP_CUDA(cudaMallocAsync(&tmp, num_er * sizeof(int2), st));
        ZP_CUDA(cudaMemcpyAsync(tmp, h.data(), num_er * sizeof(int2), cudaMemcpyHostToDevice, st));
        a.er = tmp;
        a.er_stride = 1;
      }
    }
  }
  bool aligned = true;
  for (int k = 0; k < N + 2; k++) aligned &= (reinterpret_cast<uintptr_t>(a.base[k]) & 15u) == 0;
  if (num_stripes > 1) aligned &= (stripe_stride % 16 == 0) && (parity_stride % 16 == 0);
  const uint64_t TB = zp::rs_tile_bytes(), CB = zp::rs_chunk_bytes();
  a.body_tiles = aligned ? bytes / TB : 0;
  a.tail_units_per_stripe = (bytes - a.body_tiles * TB + CB - 1) / CB;
  int dev = 0, sms = 148, occ = 1;
  ZP_CUDA(cudaGetDevice(&dev));
  ZP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const void* fn = zp::rs_kernel_ptr(recover);
  raid6c_status o = kernel_occupancy(dev, fn, zp::rs_threads() + 32, zp::rs_smem_bytes(recover), &occ);
  if (o != RAID6C_OK) return o;
  const uint64_t items = a.body_tiles * static_cast<uint64_t>(num_stripes);
  const uint64_t tail_ctas = (a.tail_units_per_stripe * static_cast<uint64_t>(num_stripes) + zp::rs_threads() - 1) /
                             zp::rs_threads();
  uint64_t grid = std::min<uint64_t>(static_cast<uint64_t>(sms) * occ, std::max<uint64_t>(items, tail_ctas));
  if (grid == 0) grid = 1;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(zp::rs_threads() + 32), args,
                                   zp::rs_smem_bytes(recover), st);
  if (tmp) cudaFreeAsync(tmp, st);
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return RAID6C_OK;
}

raid6c_status raid6c_rs_encode_strided(int N, size_t bytes, const uint8_t* data, size_t strip_stride,
                                       size_t stripe_stride, uint8_t* P, uint8_t* Q, size_t parity_stride,
                                       int num_stripes, void* stream) {
  return rs_launch(N, bytes, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, false, nullptr, 0,
                   0, static_cast<cudaStream_t>(stream));
}

raid6c_status raid6c_rs_recover_strided(int N, size_t bytes, uint8_t* data, size_t strip_stride, size_t stripe_stride,
                                        uint8_t* P, uint8_t* Q, size_t parity_stride, int num_stripes,
                                        const raid6c_erasure* erasures, int num_erasures, int erasures_on_device,
                                        void* stream) {
  return rs_launch(N, bytes, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, true, erasures,
                   num_erasures, erasures_on_device, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
