// microbench.cu -- SURVEY.md B0: the machine numbers the kernels' secondary (ALU) roofline and the
// TMA read roofline rest on, measured on this B200 instead of assumed.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o microbench tools/microbench.cu
//   ./microbench > profiles/r01_microbench.json
//
// (1) integer pipe throughput per SM per clock for the instructions the Z_p kernels are made of:
//     LOP3 (3-input logic: the XOR-accumulate with mask), SHF (funnel shift: the rotation), IADD3,
//     IMAD (integer multiply-add), each in 8 independent dependency chains per thread, 32 warps per
//     SM, cycles from clock64();
// (2) HBM read bandwidth of 1-D TMA bulk copies (cp.async.bulk, as zp_kernel issues them) from K
//     concurrent strips per CTA (K = 1, 4, 12, 58, 66: the row counts of configs 1-5), one producer
//     lane and an 8-stage mbarrier ring per CTA, two CTAs per SM, no compute -- the read ceiling
//     the stripe kernels approach; and a plain 16-byte vectorised LDG read kernel for comparison.
// Not part of the library: a standalone measurement tool.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

// ------------------------------------------------------------------ (1) integer pipes
template <int OP>
__device__ __forceinline__ void op(uint32_t& a, uint32_t b, uint32_t c) {
  if constexpr (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a) : "r"(b), "r"(c));
  if constexpr (OP == 1) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
  if constexpr (OP == 2) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
  if constexpr (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
  if constexpr (OP == 4) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
  if constexpr (OP == 5) {  // mixed stream: 1 funnel shift (ALU) + 1 multiply-add (FMA) per op pair
    asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
  }
}
template <int OP>
__global__ void alu_kernel(uint32_t* out, int iters, unsigned long long* cyc) {
  uint32_t a[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = threadIdx.x * 7 + k;
  const uint32_t b = blockIdx.x | 1u, c = threadIdx.x ^ 0x5a5a5a5au;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int k = 0; k < 8; k++) op<OP>(a[k], b + r, c);
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(cyc, t1 - t0);
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) x ^= a[k];
  if (x == 0x12345678u) out[blockIdx.x] = x;
}

// ------------------------------------------------------------------ (2) TMA bulk read streams
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int TB = 12288, ST = 8, CONS = 256;

__global__ void __launch_bounds__(CONS + 32, 2) tma_read_kernel(const uint8_t* base, uint64_t strip_stride, int K,
                                                                 uint64_t tiles, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * TB);
  uint64_t* empty = full + ST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < ST; s++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(CONS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CONS / 32) {
    if (lane == 0) {
      uint32_t stage = 0, ph = 0;
      for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int k = 0; k < K; k++) {
          asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                       ::"r"(smem_u32(&empty[stage])), "r"(ph ^ 1u) : "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[stage])), "r"(TB) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(smem + stage * TB)), "l"(base + k * strip_stride + t * TB), "r"(TB),
                       "r"(smem_u32(&full[stage])) : "memory");
          if (++stage == ST) { stage = 0; ph ^= 1u; }
        }
    }
    return;
  }
  uint32_t stage = 0, ph = 0, acc = 0;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x)
    for (int k = 0; k < K; k++) {
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                   ::"r"(smem_u32(&full[stage])), "r"(ph) : "memory");
      acc ^= reinterpret_cast<const uint32_t*>(smem + stage * TB)[tid * 12];  // touch the row
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
      if (++stage == ST) { stage = 0; ph ^= 1u; }
    }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

// ------------------------------------------------------------------ (3) TMA read K rows, bulk-store W rows
// The product kernels' memory pattern without their arithmetic: per tile, K rows in through the
// mbarrier ring, XOR-folded in registers, the fold stored to W strips (STORE: SMEM-staged bulk store or st.global from registers).
template <int STORE>  // 0: SMEM-staged bulk store, 1: st.global.v4 from registers, 2: st.global.cs.v4
__global__ void __launch_bounds__(CONS + 32, 2) tma_mix_kernel(const uint8_t* base, uint64_t strip_stride, int K,
                                                                uint8_t* obase, int W, uint64_t tiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* obuf = smem + ST * TB;
  uint64_t* full = reinterpret_cast<uint64_t*>(obuf + TB);
  uint64_t* empty = full + ST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < ST; s++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(CONS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CONS / 32) {
    if (lane == 0) {
      uint32_t stage = 0, ph = 0;
      for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int k = 0; k < K; k++) {
          asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                       ::"r"(smem_u32(&empty[stage])), "r"(ph ^ 1u) : "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[stage])), "r"(TB) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(smem + stage * TB)), "l"(base + k * strip_stride + t * TB), "r"(TB),
                       "r"(smem_u32(&full[stage])) : "memory");
          if (++stage == ST) { stage = 0; ph ^= 1u; }
        }
    }
    return;
  }
  uint32_t stage = 0, ph = 0;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    uint4 a[3] = {};
    for (int k = 0; k < K; k++) {
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}"
                   ::"r"(smem_u32(&full[stage])), "r"(ph) : "memory");
      const uint4* row = reinterpret_cast<const uint4*>(smem + stage * TB);
#pragma unroll
      for (int j = 0; j < 3; j++) {
        const uint4 v = row[tid + j * CONS];
        a[j].x ^= v.x; a[j].y ^= v.y; a[j].z ^= v.z; a[j].w ^= v.w;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
      if (++stage == ST) { stage = 0; ph ^= 1u; }
    }
    if (W == 0) {
      if ((a[0].x ^ a[1].y ^ a[2].z) == 0x9e3779b9u) obase[0] = 1;
      continue;
    }
    if (STORE != 0) {
      for (int w = 0; w < W; w++) {
        uint4* o = reinterpret_cast<uint4*>(obase + w * strip_stride + t * TB);
#pragma unroll
        for (int j = 0; j < 3; j++) {
          if (STORE == 1) o[tid + j * CONS] = a[j];
          else __stcs(o + tid + j * CONS, a[j]);
        }
      }
      continue;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(CONS) : "memory");
#pragma unroll
    for (int j = 0; j < 3; j++) reinterpret_cast<uint4*>(obuf)[tid + j * CONS] = a[j];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(CONS) : "memory");
    if (tid == 0) {
      for (int w = 0; w < W; w++)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(obase + w * strip_stride + t * TB),
                     "r"(smem_u32(obuf)), "r"(TB) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void ldg_read_kernel(const uint4* src, uint64_t n16, uint32_t* sink) {
  uint32_t acc = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  uint32_t* out;
  unsigned long long* cyc;
  CK(cudaMalloc(&out, 1 << 20));
  CK(cudaMalloc(&cyc, 8));
  printf("{\"sms\": %d, \"attr_clock_mhz\": %.0f,\n \"int_ops_per_clk_per_sm\": {", sms, clk_khz / 1e3);
  const char* names[6] = {"LOP3", "SHF.L.W", "IADD3 (2 PTX adds fused per op: counts PTX adds)", "IMAD", "IMAD.HI",
                          "SHF+IMAD mixed (counts both)"};
  const int blocks = sms * 2, threads = 512, iters = 4096;  // 32 warps per SM
  for (int o = 0; o < 6; o++) {
    float best = 0;
    for (int rep = 0; rep < 3; rep++) {
      CK(cudaMemset(cyc, 0, 8));
      if (o == 0) alu_kernel<0><<<blocks, threads>>>(out, iters, cyc);
      if (o == 1) alu_kernel<1><<<blocks, threads>>>(out, iters, cyc);
      if (o == 2) alu_kernel<2><<<blocks, threads>>>(out, iters, cyc);
      if (o == 3) alu_kernel<3><<<blocks, threads>>>(out, iters, cyc);
      if (o == 4) alu_kernel<4><<<blocks, threads>>>(out, iters, cyc);
      if (o == 5) alu_kernel<5><<<blocks, threads>>>(out, iters, cyc);
      CK(cudaDeviceSynchronize());
      unsigned long long c = 0;
      CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      const double ops_per_sm = 2.0 * threads * iters * 4.0 * 8.0 * (o == 5 ? 2 : 1);  // 2 blocks per SM
      const float v = static_cast<float>(ops_per_sm / static_cast<double>(c));
      if (v > best) best = v;
    }
    printf("%s\"%s\": %.1f", o ? ", " : "", names[o], best);
  }
  printf("},\n");
  // TMA streams
  const int Kmax = 66;
  const uint64_t tiles = 512;  // per strip: 6 MiB strips
  const uint64_t strip = tiles * TB;
  uint8_t* buf;
  CK(cudaMalloc(&buf, Kmax * strip));
  CK(cudaMemset(buf, 1, Kmax * strip));
  const size_t smem = ST * TB + 2 * ST * 8;
  CK(cudaFuncSetAttribute(tma_read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf(" \"tma_read_GBps\": {");
  const int Ks[5] = {1, 4, 12, 58, 66};
  for (int i = 0; i < 5; i++) {
    const int K = Ks[i];
    // same total bytes per point (415 MB): repeat the K strips' tiles over the whole buffer
    const uint64_t tiles_k = (Kmax * tiles) / K;
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
      CK(cudaEventRecord(e0));
      tma_read_kernel<<<sms * 2, CONS + 32, smem>>>(buf, tiles_k * TB, K, tiles_k, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    const double bytes = static_cast<double>(K) * tiles_k * TB;
    printf("%s\"K%d\": %.1f", i ? ", " : "", K, bytes / (best / 1e3) / 1e9);
  }
  printf("},\n");
  {
    float best = 1e30f;
    const uint64_t n16 = Kmax * strip / 16;
    for (int rep = 0; rep < 5; rep++) {
      CK(cudaEventRecord(e0));
      ldg_read_kernel<<<sms * 8, 512>>>(reinterpret_cast<const uint4*>(buf), n16, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf(" \"ldg128_read_GBps\": %.1f,\n", Kmax * strip / (best / 1e3) / 1e9);
  }
  {
    // read:write mixes of the configs (K strips in, W strips out per tile): 415 MB read per point
    uint8_t* obuf;
    CK(cudaMalloc(&obuf, 2 * Kmax * strip));
    const size_t msmem = ST * TB + TB + 2 * ST * 8;
    CK(cudaFuncSetAttribute(tma_mix_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem)));
    CK(cudaFuncSetAttribute(tma_mix_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem)));
    CK(cudaFuncSetAttribute(tma_mix_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(msmem)));
    const int mixes[8][2] = {{1, 1}, {2, 2}, {4, 2}, {6, 0}, {8, 2}, {12, 2}, {16, 2}, {58, 2}};
    const char* sname[3] = {"bulk_store", "st_global", "st_global_cs"};
    printf(" \"tma_read_K_store_W_GBps\": {");
    for (int m = 0; m < 3; m++) {
      printf("%s\"%s\": {", m ? ", " : "", sname[m]);
      for (int i = 0; i < 8; i++) {
        const int K = mixes[i][0], W = mixes[i][1];
        if (W == 0 && m) continue;
        const uint64_t tiles_m = (Kmax * tiles) / K;  // the whole input buffer read once, W rows per tile out
        float best = 1e30f;
        for (int rep = 0; rep < 5; rep++) {
          CK(cudaEventRecord(e0));
          if (m == 0) tma_mix_kernel<0><<<sms * 2, CONS + 32, msmem>>>(buf, tiles_m * TB, K, obuf, W, tiles_m);
          if (m == 1) tma_mix_kernel<1><<<sms * 2, CONS + 32, msmem>>>(buf, tiles_m * TB, K, obuf, W, tiles_m);
          if (m == 2) tma_mix_kernel<2><<<sms * 2, CONS + 32, msmem>>>(buf, tiles_m * TB, K, obuf, W, tiles_m);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (ms < best) best = ms;
        }
        const double bytes = static_cast<double>(K + W) * tiles_m * TB;
        printf("%s\"%d:%d\": %.1f", i ? ", " : "", K, W, bytes / (best / 1e3) / 1e9);
      }
      printf("}");
    }
    printf("},\n");
    CK(cudaFree(obuf));
  }
  printf(" \"how\": \"tools/microbench.cu: int ops = 8 independent chains x 32 warps/SM, clock64 cycles (best of 3); "
         "TMA = cp.async.bulk 12 KiB rows from K strips round-robin, 8-stage mbarrier ring, 2 CTAs/SM, no compute, "
         "415 MB read per point, best of 5 (CUDA events); K:W = the same ring + XOR fold, fold bulk-stored from SMEM or stored from registers (st.global, st.global.cs) to W strips, "
         "GB/s counts (K+W) rows per tile\"}\n");
  return 0;
}
