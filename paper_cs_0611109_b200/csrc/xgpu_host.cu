// xgpu_host.cu -- NEXT-4 entry points of libraid6c (include/raid6c.h "cross-GPU stripe layout"):
// word-range sizes, the partial-syndrome and combine+solve launches, and inter-process device
// memory (CUDA IPC) for one process per GPU.
#include <algorithm>
#include <cstring>
#include <vector>

#include "host_internal.h"

using namespace zp::host;

extern "C" {

// ---------------------------------------------------------------- NEXT-4: cross-GPU stripe layout
size_t raid6c_xgpu_range_bytes(int p, size_t bytes, int num_ranks) {
  if (!is_valid_p(p) || bytes == 0 || num_ranks < 1 || num_ranks > RAID6C_MAX_RANKS) return 0;
  const uint64_t gr = range_granule_p(p);
  const uint64_t units = (parity_bytes(p, bytes) + gr - 1) / gr;
  return static_cast<size_t>(((units + num_ranks - 1) / num_ranks) * gr);
}

// Strip table of a cross-GPU call: N+2 global-index pointers, strides.
static raid6c_status xgpu_args(raid6c_plan plan, const uint8_t* const* strips, size_t data_stride, size_t parity_stride,
                               int num_stripes, int k_lo, int k_hi, zp::ZpArgs& a) {
  if (!plan || !strips) return RAID6C_E_NULL;
  if (num_stripes < 0) return RAID6C_E_SIZE;
  if (k_lo < 0 || k_hi > plan->N + 2 || k_lo > k_hi) return RAID6C_E_INVALID_INDEX;
  for (int k = k_lo; k < k_hi; k++)
    if (!strips[k]) return RAID6C_E_NULL;
  if (num_stripes > 1 && (data_stride < plan->bytes || parity_stride < plan->pbytes)) return RAID6C_E_SIZE;
  std::memset(&a, 0, sizeof(a));
  for (int k = 0; k < plan->N + 2; k++) a.base[k] = strips[k];
  a.data_stride = data_stride;
  a.parity_stride = parity_stride;
  a.num_stripes = num_stripes;
  a.ei = plan->N;  // encode = the PQ pair
  a.ej = plan->N + 1;
  a.k_lo = k_lo;
  a.k_hi = k_hi;
  return RAID6C_OK;
}

raid6c_status raid6c_partial_strided(raid6c_plan plan, const uint8_t* const* strips, size_t data_stride,
                                     size_t parity_stride, int num_stripes, const raid6c_erasure* erasures,
                                     int num_erasures, int erasures_on_device, int k_lo, int k_hi, int num_ranges,
                                     uint8_t* const* part_p, uint8_t* const* part_q, size_t part_stride,
                                     size_t range_bytes) {
  zp::ZpArgs a;
  raid6c_status st = xgpu_args(plan, strips, data_stride, parity_stride, num_stripes, k_lo, k_hi, a);
  if (st != RAID6C_OK) return st;
  if (num_ranges < 1 || num_ranges > RAID6C_MAX_RANKS) return RAID6C_E_SIZE;
  if (!part_p || !part_q) return RAID6C_E_NULL;
  const uint64_t gr = range_granule(plan);
  if (range_bytes == 0 || range_bytes % gr != 0 || static_cast<uint64_t>(range_bytes) * num_ranges < plan->pbytes)
    return RAID6C_E_SIZE;
  if (num_stripes > 1 && part_stride < range_bytes) return RAID6C_E_SIZE;
  const int used = static_cast<int>((plan->pbytes + range_bytes - 1) / range_bytes);  // ranges holding bytes
  for (int g = 0; g < used; g++)
    if (!part_p[g] || !part_q[g]) return RAID6C_E_NULL;
  for (int g = 0; g < num_ranges; g++) {
    a.part_p[g] = part_p[g];
    a.part_q[g] = part_q[g];
  }
  a.nranges = used;
  a.range_bytes = range_bytes;
  a.part_stride = part_stride;
  DeviceGuard g(plan->device);
  if (erasures) {
    st = set_erasures(plan, a, erasures, num_erasures, erasures_on_device, num_stripes, false);
    if (st != RAID6C_OK) return st;
  }
  return launch(plan, a, zp::KMODE_PARTIAL, plan->stream);
}

raid6c_status raid6c_combine_strided(raid6c_plan plan, uint8_t* const* strips, size_t data_stride,
                                     size_t parity_stride, int num_stripes, const raid6c_erasure* erasures,
                                     int num_erasures, int erasures_on_device, int num_sources,
                                     const uint8_t* const* src_p, const uint8_t* const* src_q, size_t part_stride,
                                     size_t range_lo, size_t range_hi) {
  zp::ZpArgs a;
  raid6c_status st = xgpu_args(plan, strips, data_stride, parity_stride, num_stripes, 0, 0, a);
  if (st != RAID6C_OK) return st;
  if (num_sources < 1 || num_sources > RAID6C_MAX_RANKS) return RAID6C_E_SIZE;
  if (!src_p || !src_q) return RAID6C_E_NULL;
  for (int r = 0; r < num_sources; r++) {
    if (!src_p[r] || !src_q[r]) return RAID6C_E_NULL;
    a.src_p[r] = src_p[r];
    a.src_q[r] = src_q[r];
  }
  const uint64_t gr = range_granule(plan);
  // both ends on the range grid (or the end of the strip): the kernels work in whole tiles /
  // groups up to range_hi rounded up, which must not reach into the next owner's range
  if (range_lo % gr != 0 || range_hi < range_lo || range_hi > plan->pbytes ||
      (range_hi % gr != 0 && range_hi != plan->pbytes))
    return RAID6C_E_SIZE;
  if (num_stripes > 1 && part_stride < range_hi - range_lo) return RAID6C_E_SIZE;
  a.nsrc = num_sources;
  a.range_lo = range_lo;
  a.range_hi = range_hi;
  a.part_stride = part_stride;
  DeviceGuard g(plan->device);
  if (erasures) {
    st = set_erasures(plan, a, erasures, num_erasures, erasures_on_device, num_stripes, true);
    if (st != RAID6C_OK) return st;
  }
  // output strips of every stripe must be present: check against the (host-known) pairs
  if (!erasures || !erasures_on_device) {
    for (int s = 0; s < (erasures ? num_erasures : 1); s++) {
      const int x = erasures ? std::min(erasures[s].lost_i, erasures[s].lost_j) : plan->N;
      const int y = erasures ? std::max(erasures[s].lost_i, erasures[s].lost_j) : plan->N + 1;
      if (!strips[x] || !strips[y]) return RAID6C_E_NULL;
    }
  }
  return launch_combine(plan, a, plan->stream);
}

raid6c_status raid6c_dev_alloc(size_t bytes, int device, void** dev_ptr) {
  if (!dev_ptr) return RAID6C_E_NULL;
  *dev_ptr = nullptr;
  if (bytes == 0) return RAID6C_E_SIZE;
  DeviceGuard g(device);
  ZP_CUDA(cudaMalloc(dev_ptr, bytes));
  return RAID6C_OK;
}

raid6c_status raid6c_dev_free(void* dev_ptr) {
  if (!dev_ptr) return RAID6C_E_NULL;
  ZP_CUDA(cudaFree(dev_ptr));
  return RAID6C_OK;
}

raid6c_status raid6c_ipc_export(const void* dev_ptr, uint8_t handle[64]) {
  if (!dev_ptr || !handle) return RAID6C_E_NULL;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
  cudaIpcMemHandle_t h;
  ZP_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  std::memcpy(handle, &h, 64);
  return RAID6C_OK;
}

raid6c_status raid6c_ipc_open(const uint8_t handle[64], int device, void** dev_ptr) {
  if (!handle || !dev_ptr) return RAID6C_E_NULL;
  *dev_ptr = nullptr;
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  ZP_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return RAID6C_OK;
}

raid6c_status raid6c_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return RAID6C_E_NULL;
  ZP_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return RAID6C_OK;
}

}  // extern "C"
