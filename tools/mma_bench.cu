// Microbenchmark: cycles per tcgen05.mma kind::tf32 (M=128) for SS and TS
// operand placement and several N, issued back to back by one thread on every
// SM. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//            -I paper_1709_07175_b200/csrc tools/mma_bench.cu -o mma_bench
#include <cstdio>

#include "tc_util.cuh"

using namespace lpca::tc;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = idesc_tf32(128, N, 0, 0);
  const uint64_t da = sw128_desc(smem_u32(smem), 16, 1024);
  const uint64_t db = sw128_desc(smem_u32(smem) + 16384, 16, 1024);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (TS)
        mma_tf32_ts(tmem, tmem + 256, db, idesc, 1u);
      else
        mma_tf32(tmem, da, db, idesc, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// Pair (cta_group::2, M = 256) variant: rank 0 issues, both CTAs hold A (TMEM) and half of B.
template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) bench2(long long* out, int iters) {
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
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = idesc_tf32(256, N, 0, 0);
  const uint64_t da = sw128_desc(smem_u32(smem), 16, 1024);
  const uint64_t db = sw128_desc(smem_u32(smem) + 16384, 16, 1024);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    if (rank == 0) {
      for (int it = 0; it < iters; ++it) {
        if (TS)
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
              "r"(tmem + 256), "l"(db), "r"(idesc), "r"(1u)
              : "memory");
        else
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(1u)
              : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"(static_cast<uint16_t>(3))
          : "memory");
    }
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

template <int N, bool TS>
void run2(long long* d, int sms) {
  const int iters = 4096;
  cudaFuncSetAttribute(bench2<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  bench2<N, TS><<<sms, 128, 65536 + 1024>>>(d, iters);
  bench2<N, TS><<<sms, 128, 65536 + 1024>>>(d, iters);
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; i += 2) avg += h[i];
  avg /= sms / 2;
  printf("pair %s M=256 N=%3d: %.1f cycles/MMA (1-SM M=128 floor 128*N/256 = %d)\n", TS ? "TS" : "SS", N,
         avg / iters, 128 * N / 256);
}

template <int N, bool TS>
void run(long long* d, int sms) {
  const int iters = 4096;
  cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  bench<N, TS><<<sms, 128, 65536 + 1024>>>(d, iters);
  bench<N, TS><<<sms, 128, 65536 + 1024>>>(d, iters);
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("%s N=%3d: %.1f cycles/MMA (floor 128*N/256 = %d)\n", TS ? "TS" : "SS", N, avg / iters, 128 * N / 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  int sms = 148;
  run<64, false>(d, sms);
  run<112, false>(d, sms);
  run<128, false>(d, sms);
  run<224, false>(d, sms);
  run<256, false>(d, sms);
  run<64, true>(d, sms);
  run<112, true>(d, sms);
  run<128, true>(d, sms);
  run<224, true>(d, sms);
  run<256, true>(d, sms);
  run<16, true>(d, sms);
  run2<16, false>(d, sms);
  run2<16, true>(d, sms);
  run2<64, true>(d, sms);
  run2<112, false>(d, sms);
  run2<112, true>(d, sms);
  run2<128, true>(d, sms);
  run2<224, true>(d, sms);
  run2<256, true>(d, sms);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
