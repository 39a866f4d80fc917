// host_pipeline.cu -- the host-buffer (end-to-end) path of libraid6c: stripes stream through the
// plan's device staging ring, H2D copy, kernel and D2H copy of successive chunks overlapping on
// three streams (raid6c_encode_host / raid6c_recover_host, include/raid6c.h).
#include <algorithm>
#include <cstring>
#include <vector>

#include "host_internal.h"

namespace zp {
namespace host {

// ------------------------------------------------------------------ host-buffer pipeline
raid6c_status host_setup(raid6c_plan pl, int num_stripes) {
  DeviceGuard g(pl->device);
  const size_t sd = (pl->bytes + 255) / 256 * 256, sp = (pl->pbytes + 255) / 256 * 256;
  const size_t stripe_dev = static_cast<size_t>(pl->N) * sd + 2 * sp;
  const size_t target = size_t(512) << 20;
  int cs = static_cast<int>(std::max<size_t>(1, target / stripe_dev));
  cs = std::min(cs, std::max(1, num_stripes));
  const size_t need = static_cast<size_t>(cs) * stripe_dev;
  if (!pl->host_ready) {
    for (int i = 0; i < 3; i++) ZP_CUDA(cudaStreamCreateWithFlags(&pl->hs[i], cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++) {
      ZP_CUDA(cudaEventCreateWithFlags(&pl->ev_in[i], cudaEventDisableTiming));
      ZP_CUDA(cudaEventCreateWithFlags(&pl->ev_k[i], cudaEventDisableTiming));
      ZP_CUDA(cudaEventCreateWithFlags(&pl->ev_out[i], cudaEventDisableTiming));
    }
    pl->host_ready = true;
  }
  if (pl->slot_bytes < need || pl->slot_stripes < cs) {
    if (pl->d_stage) {
      ZP_CUDA(cudaDeviceSynchronize());
      cudaFree(pl->d_stage);
      pl->d_stage = nullptr;
    }
    ZP_CUDA(cudaMalloc(&pl->d_stage, 2 * need));
    pl->slot_bytes = need;
    pl->slot_stripes = cs;
  }
  return RAID6C_OK;
}

// Copy `rows` strips of `width` bytes: host rows at src + r*spitch -> device rows at dst + r*dpitch.
raid6c_status copy_rows(uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width, int rows,
                        cudaMemcpyKind kind, cudaStream_t st) {
  if (rows <= 0) return RAID6C_OK;
  if (rows == 1) {
    ZP_CUDA(cudaMemcpyAsync(dst, src, width, kind, st));
  } else {
    ZP_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, st));
  }
  return RAID6C_OK;
}

raid6c_status host_run(raid6c_plan pl, uint8_t* data, size_t strip_stride, size_t stripe_stride, uint8_t* P,
                       uint8_t* Q, size_t parity_stride, int num_stripes, const raid6c_erasure* er,
                       int num_erasures, bool recover) {
  if (!pl) return RAID6C_E_NULL;
  if (num_stripes < 0) return RAID6C_E_SIZE;
  if (num_stripes == 0) return RAID6C_OK;
  if (!data || !P || !Q) return RAID6C_E_NULL;
  if (pl->N > 1 && strip_stride < pl->bytes) return RAID6C_E_SIZE;
  if (num_stripes > 1 && (stripe_stride < pl->bytes || parity_stride < pl->pbytes)) return RAID6C_E_SIZE;
  std::vector<int2> pairs;
  if (recover) {
    if (!er) return RAID6C_E_NULL;
    if (num_erasures != 1 && num_erasures != num_stripes) return RAID6C_E_SIZE;
    pairs.resize(num_stripes);
    for (int s = 0; s < num_stripes; s++) {
      raid6c_erasure e = er[num_erasures == 1 ? 0 : s];
      pair_of_single(pl->N, e.lost_i, e.lost_j);
      raid6c_status c = check_erasure(pl->N, e.lost_i, e.lost_j);
      if (c != RAID6C_OK) return c;
      pairs[s] = make_int2(std::min(e.lost_i, e.lost_j), std::max(e.lost_i, e.lost_j));
    }
  }
  raid6c_status st = host_setup(pl, num_stripes);
  if (st != RAID6C_OK) return st;
  DeviceGuard g(pl->device);
  const int N = pl->N;
  const size_t sd = (pl->bytes + 255) / 256 * 256, sp = (pl->pbytes + 255) / 256 * 256;
  const int cs = pl->slot_stripes;
  cudaStream_t s_in = pl->hs[0], s_k = pl->hs[1], s_out = pl->hs[2];
  if (recover) {
    // per-stripe pairs for the whole call, uploaded once on the kernel stream
    std::vector<raid6c_erasure> ev(num_stripes);
    for (int s = 0; s < num_stripes; s++) ev[s] = {pairs[s].x, pairs[s].y};
    st = upload_erasures(pl, ev.data(), num_stripes, s_k);
    if (st != RAID6C_OK) return st;
  }
  // order after anything already queued on the plan stream
  ZP_CUDA(cudaEventRecord(pl->ev_out[0], pl->stream));
  ZP_CUDA(cudaStreamWaitEvent(s_in, pl->ev_out[0], 0));
  ZP_CUDA(cudaEventRecord(pl->ev_out[1], pl->stream));
  uint64_t h2d = 0, d2h = 0;
  int c = 0;
  for (int s0 = 0; s0 < num_stripes; s0 += cs, c++) {
    const int slot = c & 1;
    const int ns = std::min(cs, num_stripes - s0);
    uint8_t* base = pl->d_stage + static_cast<size_t>(slot) * pl->slot_bytes;
    uint8_t* dP = base + static_cast<size_t>(cs) * N * sd;
    uint8_t* dQ = dP + static_cast<size_t>(cs) * sp;
    const size_t dstripe = static_cast<size_t>(N) * sd;
    if (c >= 2) ZP_CUDA(cudaStreamWaitEvent(s_in, pl->ev_out[slot], 0));
    // ---- H2D of the inputs
    for (int i = 0; i < ns; i++) {
      const int s = s0 + i;
      const uint8_t* hd = data + static_cast<size_t>(s) * stripe_stride;
      uint8_t* dd = base + static_cast<size_t>(i) * dstripe;
      int x = N, y = N + 1;
      if (recover) { x = pairs[s].x; y = pairs[s].y; }
      // contiguous runs of surviving data strips
      int k = 0;
      while (k < N) {
        if (k == x || k == y) { k++; continue; }
        int e = k;
        while (e < N && e != x && e != y) e++;
        st = copy_rows(dd + static_cast<size_t>(k) * sd, sd, hd + static_cast<size_t>(k) * strip_stride, strip_stride,
                       pl->bytes, e - k, cudaMemcpyHostToDevice, s_in);
        if (st != RAID6C_OK) return st;
        h2d += static_cast<uint64_t>(e - k) * pl->bytes;
        k = e;
      }
      if (recover && x != N && y != N) {
        ZP_CUDA(cudaMemcpyAsync(dP + static_cast<size_t>(i) * sp, P + static_cast<size_t>(s) * parity_stride, pl->pbytes,
                                cudaMemcpyHostToDevice, s_in));
        h2d += pl->pbytes;
      }
      if (recover && y != N + 1) {
        ZP_CUDA(cudaMemcpyAsync(dQ + static_cast<size_t>(i) * sp, Q + static_cast<size_t>(s) * parity_stride, pl->pbytes,
                                cudaMemcpyHostToDevice, s_in));
        h2d += pl->pbytes;
      }
    }
    ZP_CUDA(cudaEventRecord(pl->ev_in[slot], s_in));
    // ---- kernel
    ZP_CUDA(cudaStreamWaitEvent(s_k, pl->ev_in[slot], 0));
    zp::ZpArgs a;
    std::memset(&a, 0, sizeof(a));
    for (int k = 0; k < N; k++) a.base[k] = base + static_cast<size_t>(k) * sd;
    a.base[N] = dP;
    a.base[N + 1] = dQ;
    a.data_stride = dstripe;
    a.parity_stride = sp;
    a.num_stripes = ns;
    a.ei = N;
    a.ej = N + 1;
    if (recover) {
      a.er = pl->d_er + s0;
      a.er_stride = 1;
      if (pl->ext) a.prog = pl->d_prog;
    }
    st = launch(pl, a, recover ? zp::KMODE_RECOVER : zp::KMODE_ENCODE, s_k);
    if (st != RAID6C_OK) return st;
    ZP_CUDA(cudaEventRecord(pl->ev_k[slot], s_k));
    // ---- D2H of the outputs
    ZP_CUDA(cudaStreamWaitEvent(s_out, pl->ev_k[slot], 0));
    if (!recover) {
      st = copy_rows(P + static_cast<size_t>(s0) * parity_stride, parity_stride, dP, sp, pl->pbytes, ns,
                     cudaMemcpyDeviceToHost, s_out);
      if (st != RAID6C_OK) return st;
      st = copy_rows(Q + static_cast<size_t>(s0) * parity_stride, parity_stride, dQ, sp, pl->pbytes, ns,
                     cudaMemcpyDeviceToHost, s_out);
      if (st != RAID6C_OK) return st;
      d2h += 2ull * ns * pl->pbytes;
    } else {
      for (int i = 0; i < ns; i++) {
        const int s = s0 + i;
        const int lost[2] = {pairs[s].x, pairs[s].y};
        for (int q = 0; q < 2; q++) {
          const int k = lost[q];
          if (k < N) {
            ZP_CUDA(cudaMemcpyAsync(data + static_cast<size_t>(s) * stripe_stride + static_cast<size_t>(k) * strip_stride,
                                    base + static_cast<size_t>(i) * dstripe + static_cast<size_t>(k) * sd, pl->bytes,
                                    cudaMemcpyDeviceToHost, s_out));
            d2h += pl->bytes;
          } else {
            uint8_t* hdst = (k == N ? P : Q) + static_cast<size_t>(s) * parity_stride;
            const uint8_t* dsrc = (k == N ? dP : dQ) + static_cast<size_t>(i) * sp;
            ZP_CUDA(cudaMemcpyAsync(hdst, dsrc, pl->pbytes, cudaMemcpyDeviceToHost, s_out));
            d2h += pl->pbytes;
          }
        }
      }
    }
    ZP_CUDA(cudaEventRecord(pl->ev_out[slot], s_out));
  }
  ZP_CUDA(cudaStreamSynchronize(s_out));
  ZP_CUDA(cudaStreamSynchronize(s_k));
  ZP_CUDA(cudaGetLastError());
  pl->h2d = h2d;
  pl->d2h = d2h;
  return RAID6C_OK;
}

}  // namespace host
}  // namespace zp

using namespace zp::host;

extern "C" {

raid6c_status raid6c_encode_host(raid6c_plan plan, const uint8_t* data, size_t strip_stride, size_t stripe_stride,
                                 uint8_t* P, uint8_t* Q, size_t parity_stride, int num_stripes) {
  return host_run(plan, const_cast<uint8_t*>(data), strip_stride, stripe_stride, P, Q, parity_stride, num_stripes,
                  nullptr, 0, false);
}

raid6c_status raid6c_recover_host(raid6c_plan plan, uint8_t* data, size_t strip_stride, size_t stripe_stride,
                                  uint8_t* P, uint8_t* Q, size_t parity_stride, int num_stripes,
                                  const raid6c_erasure* erasures, int num_erasures) {
  return host_run(plan, data, strip_stride, stripe_stride, P, Q, parity_stride, num_stripes, erasures, num_erasures,
                  true);
}

raid6c_status raid6c_host_traffic(raid6c_plan plan, uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  if (!plan || !h2d_bytes || !d2h_bytes) return RAID6C_E_NULL;
  *h2d_bytes = plan->h2d;
  *d2h_bytes = plan->d2h;
  return RAID6C_OK;
}

}  // extern "C"
