// Probe: kind::f16 MMA with A in TMEM (TS form) — which TMEM packing of fp16 A
// (two K-consecutive values per 32-bit column, low half = even k) gives D = A B^T?
// B: N x K fp16, K-major, SWIZZLE_128B (64 halves per 128 B row), K = 16 per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_1709_07175_b200/csrc \
//        tools/f16_ts_probe.cu -o tools/f16_ts_probe
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "tc_util.cuh"

using namespace lpca::tc;
constexpr int M = 128, N = 64, K = 64;  // K = 64: four K=16 MMAs over one 128 B swizzle row

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__global__ void probe(const __half* a, const __half* b, float* d, int ts) {
  __shared__ __align__(1024) uint8_t sb[N * 128];
  __shared__ __align__(1024) uint8_t sa[M * 128];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int t = threadIdx.x;
  if (t < 32) tmem_alloc(&slot, 256);
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  // B and A (for SS) rows into SW128 layout: row r, 16 B chunk c at (c ^ (r & 7))
  for (int r = t; r < N; r += blockDim.x)
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4*>(sb + r * 128 + ((c ^ (r & 7)) << 4)) =
          *reinterpret_cast<const uint4*>(b + r * K + c * 8);
  for (int r = t; r < M; r += blockDim.x)
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4*>(sa + r * 128 + ((c ^ (r & 7)) << 4)) =
          *reinterpret_cast<const uint4*>(a + r * K + c * 8);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  // A into TMEM columns 128.. : lane = row, column c holds (k = 2c, 2c+1) packed, low = even
  {
    const int row = t;  // 128 threads, warp w owns lanes 32w..
    float v[32];
    for (int c = 0; c < 32; ++c) {
      __half2 h = __halves2half2(a[row * K + 2 * c], a[row * K + 2 * c + 1]);
      v[c] = *reinterpret_cast<float*>(&h);
    }
    tmem_st32(tm + ((static_cast<uint32_t>(t / 32) * 32) << 16) + 128, v);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint64_t db = sw128_desc(smem_u32(sb), 16, 1024);
    const uint64_t da = sw128_desc(smem_u32(sa), 16, 1024);
    for (int kk = 0; kk < K / 16; ++kk) {
      if (ts)
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm),
            "r"(tm + 128 + kk * 8), "l"(db + 2 * kk), "r"(idesc_f16(M, N)), "r"(kk > 0 ? 1u : 0u)
            : "memory");
      else
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
            "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(idesc_f16(M, N)), "r"(kk > 0 ? 1u : 0u)
            : "memory");
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tm + ((static_cast<uint32_t>(t / 32) * 32) << 16) + c0, v);
    for (int e = 0; e < 16; ++e) d[t * N + c0 + e] = v[e];
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_dealloc(tm, 256);
}

int main() {
  __half *a, *b;
  float* d;
  cudaMallocManaged(&a, M * K * sizeof(__half));
  cudaMallocManaged(&b, N * K * sizeof(__half));
  cudaMallocManaged(&d, M * N * sizeof(float));
  srand(1);
  for (int i = 0; i < M * K; ++i) a[i] = __float2half(static_cast<float>(rand() % 7 - 3));
  for (int i = 0; i < N * K; ++i) b[i] = __float2half(static_cast<float>(rand() % 7 - 3));
  for (int ts = 0; ts < 2; ++ts) {
    probe<<<1, 128>>>(a, b, d, ts);
    cudaError_t e = cudaDeviceSynchronize();
    double err = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        float s = 0;
        for (int k = 0; k < K; ++k) s += __half2float(a[i * K + k]) * __half2float(b[j * K + k]);
        err = fmax(err, fabs(s - d[i * N + j]));
      }
    printf("%s: %s max |err| = %g (d[0]=%g)\n", ts ? "TS" : "SS", cudaGetErrorString(e), err, d[0]);
  }
  return 0;
}
