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
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
