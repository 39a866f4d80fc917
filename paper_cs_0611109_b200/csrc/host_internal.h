// host_internal.h -- internals shared by the host-side translation units of libraid6c
// (raid6c_host.cu: plans, launch, the core C ABI; host_pipeline.cu: the host-buffer path;
// xgpu_host.cu: NEXT-4; rs_host.cu: NEXT-3).  Not part of the public ABI (include/raid6c.h).
#pragma once
#include <atomic>
#include <memory>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "raid6c.h"
#include "zp_args.h"

namespace zp {
cudaError_t harness_fill(uint8_t* dst, uint64_t strip_stride, uint64_t stripe_stride, uint64_t len, int nstrips,
                         int nstripes, uint64_t seed, int cfg, int stripe0, int strip0, int sparse_mode,
                         cudaStream_t st);
cudaError_t harness_count_mismatch(const uint8_t* a, const uint8_t* b, uint64_t len, uint64_t* out, cudaStream_t st);
cudaError_t harness_digest(const uint8_t* src, uint64_t strip_stride, uint64_t stripe_stride, uint64_t len,
                           int nstrips, int nstripes, uint64_t* out, cudaStream_t st);
// NEXT-3 Reed-Solomon baseline (rs.cu)
const void* rs_kernel_ptr(bool recover);
size_t rs_smem_bytes(bool recover);
int rs_tile_bytes();
int rs_chunk_bytes();
int rs_threads();
}  // namespace zp

struct raid6c_plan_s {
  int p = 0, N = 0;
  size_t bytes = 0, pbytes = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  const zp::FastEntry* fe = nullptr;
  int num_sms = 148;
  int occ[7] = {1, 1, 1, 1, 1, 1, 1};  // CTAs per SM per kernel mode
  bool ext = false;           // N > p: extended code of Eq. (qext)
  std::mutex mu;              // serialises the shared single-stripe plans' program buffer
  zp::ExtProg* d_prog = nullptr;
  size_t prog_cap = 0;
  int2* d_er = nullptr;
  size_t er_cap = 0;
  // d_er / d_prog are rewritten by later calls, possibly on another stream (plan_set_stream):
  // the last launch that reads them records this event, and every rewrite waits for it
  cudaEvent_t tables_done = nullptr;
  bool tables_pending = false;
  raid6c_status sticky = RAID6C_OK;
  // host-buffer pipeline
  uint8_t* d_stage = nullptr;
  size_t slot_bytes = 0;
  int slot_stripes = 0;
  cudaStream_t hs[3] = {nullptr, nullptr, nullptr};  // in, kernel, out
  cudaEvent_t ev_in[2] = {}, ev_k[2] = {}, ev_out[2] = {};
  bool host_ready = false;
  uint64_t h2d = 0, d2h = 0;
};

namespace zp {
namespace host {

extern std::atomic<uint64_t> g_launches;  // kernels launched through the library (all plans)
extern thread_local std::string g_last_err;

raid6c_status cuda_fail(cudaError_t e);
#define ZP_CUDA(call)                              \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_);   \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

bool is_valid_p(int p);
size_t word_count(int p, size_t bytes);
size_t parity_bytes(int p, size_t bytes);
bool ext_supported_p(int p);
raid6c_status kernel_occupancy(int device, const void* fn, int threads, size_t smem, int* occ);
raid6c_status plan_init(raid6c_plan pl, int p, int N, size_t bytes, int device, cudaStream_t stream);
void plan_release(raid6c_plan pl);
// Launch one batch of plan pl's kernel for `mode` (zp::KMODE_*); a.base / strides / erasures set.
raid6c_status launch(raid6c_plan pl, zp::ZpArgs& a, int mode, cudaStream_t st);
raid6c_status launch_combine(raid6c_plan pl, zp::ZpArgs& a, cudaStream_t st);
raid6c_status check_erasure(int N, int i, int j);
void pair_of_single(int N, int i, int& j);  // lost_j == RAID6C_NONE -> the pair the library runs
raid6c_status strided_args(raid6c_plan pl, const uint8_t* data, size_t strip_stride, size_t stripe_stride,
                           const uint8_t* P, const uint8_t* Q, size_t parity_stride, int num_stripes,
                           zp::ZpArgs& a);
uint64_t range_granule_p(int p);
uint64_t range_granule(raid6c_plan pl);
raid6c_status upload_erasures(raid6c_plan pl, const raid6c_erasure* er, int count, cudaStream_t st);
raid6c_status set_erasures(raid6c_plan plan, zp::ZpArgs& a, const raid6c_erasure* erasures, int num_erasures,
                           int erasures_on_device, int num_stripes, bool with_programs);
raid6c_status cached_plan(int p, int N, size_t bytes, std::shared_ptr<raid6c_plan_s>* out);
raid6c_status host_run(raid6c_plan pl, uint8_t* data, size_t strip_stride, size_t stripe_stride, uint8_t* P,
                       uint8_t* Q, size_t parity_stride, int num_stripes, const raid6c_erasure* er, int num_er,
                       bool recover);

}  // namespace host
}  // namespace zp
