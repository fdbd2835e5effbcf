// Throughput of the converter's instruction mix on one SM: F2FP (fp32 pair ->
// half2), FMUL, LOP3 — warp-instructions per cycle per SM for 1..8 warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cvt_bench tools/cvt_bench.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

template <int kOp>
__global__ void bench(float* out, int iters, long long* cyc) {
  float a[16];
  for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 0.001f + j;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      if (kOp == 0) {  // F2FP pack
        __half2 h = __floats2half2_rn(a[j], a[j + 1]);
        acc ^= *reinterpret_cast<uint32_t*>(&h);
        a[j] += 1.0f;  // keep inputs changing (FADD)
      } else if (kOp == 1) {  // FMUL only
        a[j] = a[j] * 1.0001f;
        a[j + 1] = a[j + 1] * 0.9999f;
      } else {  // LOP only
        acc += __float_as_uint(a[j]) & 0xffffe000u;
        a[j] = __uint_as_float(__float_as_uint(a[j]) ^ 1u);
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
  for (int j = 0; j < 16; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  const int iters = 4096;
  const char* names[3] = {"F2FP pack (+1 FADD)", "FMUL x2", "LOP + IADD/LOP x2"};
  for (int op = 0; op < 3; ++op)
    for (int warps : {1, 4, 8, 16}) {
      if (op == 0) bench<0><<<1, 32 * warps>>>(out, iters, cyc);
      if (op == 1) bench<1><<<1, 32 * warps>>>(out, iters, cyc);
      if (op == 2) bench<2><<<1, 32 * warps>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      const double per_inner = double(cyc[0]) / iters / 8;  // cycles per j-step (one pack)
      printf("%-22s warps %2d: %.2f cyc per step per warp-group -> %.2f steps/clk/SM (warp-level)\n", names[op], warps,
             per_inner, warps / per_inner);
    }
  return 0;
}
