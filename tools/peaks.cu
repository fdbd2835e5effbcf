// Roofline denominators the bench line divides by (BASELINE.md §4 asks for them):
// sustained dense throughput of the units the X passes and the l x l step run on,
// measured on every SM for ~2 s each (long enough to reach the power-capped
// clock a full bench step runs at), timed with CUDA events.
//   f16   : tcgen05.mma.cta_group::2.kind::f16, M = 256, N = 256, K = 16, A from
//           TMEM (the TS form the X passes issue), fp32 accumulate
//   tf32  : the same with kind::tf32 (K = 8)
//   dmma  : mma.sync m8n8k4 f64 (the fp64 tensor path of gemm_simt.cu)
//   dfma  : dependent-free DFMA chains on every lane
// Prints one JSON object. Build + run: python tools/peaks.py (writes profiles/peaks_r02.json).
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_util.cuh"

using namespace lpca::tc;

__host__ __device__ constexpr uint32_t idesc_f16_(int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

template <bool F16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair_mma(long long* cycles, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.0f;
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = F16 ? idesc_f16_(256, 256) : idesc_tf32(256, 256, 0, 0);
  const uint64_t db = sw128_desc(smem_u32(smem), 16, 1024);
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    if (rank == 0) {
      for (int it = 0; it < iters; ++it) {
        if (F16)
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
              "r"(tmem + 256), "l"(db), "r"(idesc), "r"(1u)
              : "memory");
        else
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
              "r"(tmem + 256), "l"(db), "r"(idesc), "r"(1u)
              : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"(static_cast<uint16_t>(3))
          : "memory");
    }
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

__global__ void __launch_bounds__(256) dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void __launch_bounds__(256) dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j] = j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = fma(c[j], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 12345.678) out[0] = s;
}

struct Res {
  double tflops, mhz;
};

template <typename L>
Res timed(L launch, double flops_per_launch, long long* dcyc, int nblk, double seconds) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms1 = 0;
  cudaEventElapsedTime(&ms1, e0, e1);
  int reps = static_cast<int>(seconds * 1e3 / (ms1 > 1e-3 ? ms1 : 1e-3));
  if (reps < 1) reps = 1;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  Res res{flops_per_launch * reps / (ms * 1e-3) / 1e12, 0.0};
  if (dcyc) {
    long long h[512];
    cudaMemcpy(h, dcyc, sizeof(long long) * nblk, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < nblk; ++i) avg += static_cast<double>(h[i]);
    res.mhz = avg / nblk / (ms * 1e-3 / reps) / 1e6;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return res;
}

int main() {
  int sms = 0, dev = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long* dcyc;
  double* dout;
  cudaMalloc(&dcyc, 512 * sizeof(long long));
  cudaMalloc(&dout, 64);
  const int pairs = sms / 2;
  const int it_mma = 1 << 16;
  cudaFuncSetAttribute(pair_mma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  cudaFuncSetAttribute(pair_mma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  // per pair instruction: 2 * 256 * 256 * K flops (K = 16 f16, 8 tf32)
  const Res f16 = timed([&] { pair_mma<true><<<2 * pairs, 128, 32768 + 1024>>>(dcyc, it_mma); },
                        2.0 * 256 * 256 * 16 * it_mma * pairs, dcyc, 2 * pairs, 2.0);
  const Res tf32 = timed([&] { pair_mma<false><<<2 * pairs, 128, 32768 + 1024>>>(dcyc, it_mma); },
                         2.0 * 256 * 256 * 8 * it_mma * pairs, dcyc, 2 * pairs, 2.0);
  const int it_d = 1 << 14, blocks = sms * 4;
  const Res dm = timed([&] { dmma<<<blocks, 256>>>(dout, it_d); },
                       2.0 * 8 * 8 * 4 * 8.0 * it_d * blocks * (256 / 32), nullptr, 0, 2.0);
  const Res df = timed([&] { dfma<<<blocks, 256>>>(dout, it_d); }, 2.0 * 8 * it_d * blocks * 256.0, nullptr, 0, 2.0);
  const cudaError_t err = cudaDeviceSynchronize();
  printf("{\"f16_tcgen05_tflops\": %.1f, \"f16_sm_mhz\": %.0f, \"tf32_tcgen05_tflops\": %.1f, \"tf32_sm_mhz\": %.0f, "
         "\"dmma_f64_tflops\": %.2f, \"dfma_f64_tflops\": %.2f, \"sms\": %d, \"error\": \"%s\"}\n",
         f16.tflops, f16.mhz, tf32.tflops, tf32.mhz, dm.tflops, df.tflops, sms, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
