// DFMA / DADD / DMUL issue rate per SM (fp64 pipe), measured with clock64 on
// one CTA and a full grid: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dfma_bench.cu -o tools/dfma_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_loop(double* out, long long* cyc, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) x[j] = threadIdx.x * 1e-3 + j;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = fma(x[j], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void dfma_latency(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void div_latency(double* out, long long* cyc, int iters, double a) {
  double x = threadIdx.x + 1.5;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = a / x + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void shfl_latency(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void bar_latency(double* out, long long* cyc, int iters) {
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = 0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  long long h[148];
  const int iters = 4096;
  for (int threads : {32, 128, 256, 1024}) {
    dfma_loop<8><<<1, threads>>>(out, cyc, iters, 0.999, 1e-3);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("1 CTA %4d thr: %.2f DFMA lanes/clk/SM\n", threads, double(threads) * iters * 8 / h[0]);
  }
  dfma_loop<8><<<148, 1024>>>(out, cyc, iters, 0.999, 1e-3);
  cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
  printf("148 CTAs x 1024: %.2f DFMA lanes/clk/SM\n", 1024.0 * iters * 8 / h[0]);
  dfma_latency<<<1, 32>>>(out, cyc, iters, 0.999, 1e-3);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f clk\n", double(h[0]) / iters);
  div_latency<<<1, 32>>>(out, cyc, iters, 0.999);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("fp64 div + add dependent latency: %.1f clk\n", double(h[0]) / iters);
  shfl_latency<<<1, 32>>>(out, cyc, iters);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("fp64 shfl + add dependent latency: %.1f clk\n", double(h[0]) / iters);
  for (int threads : {256, 1024}) {
    bar_latency<<<1, threads>>>(out, cyc, iters);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads %d thr: %.1f clk\n", threads, double(h[0]) / iters);
  }
  return 0;
}
