// TMA streaming roofline for the X-pass tile shapes: a persistent kernel (one
// CTA per SM) that only moves X (m x n fp32, row-major) into shared memory
// through a ring of tiles, with the tile shapes the pass kernels use.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1709_07175_b200/csrc \
//        tools/tma_stream.cu -o tools/tma_stream -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>

#include "tc_util.cuh"

using namespace lpca::tc;

struct Shape {
  const char* name;
  int box_inner, box_outer;  // elements (cols), rows
  int loads;                 // boxes per stage (side by side along columns)
  bool swz;
  bool row_tiles;            // XW: a CTA walks columns of a row block; XTU: rows of a column block
};

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int m, int n, Shape sh,
                                                int stages) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = sh.box_inner * sh.box_outer * 4;
  const int stage_bytes = box_bytes * sh.loads;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // tiles: XW = (row block of box_outer rows) x (column step of box_inner*loads)
  //        XTU = (column block of box_inner) x (row step of box_outer)
  // XTU: items = column blocks x row chunks (chunk-major, ~8 per CTA), as the pass kernel
  const int ntiles = n / sh.box_inner;
  const int chunks = (8 * gridDim.x + ntiles - 1) / ntiles;
  const int chunk_rows = ((m + chunks - 1) / chunks + sh.box_outer - 1) / sh.box_outer * sh.box_outer;
  const long tile_a = sh.row_tiles ? (m + sh.box_outer - 1) / sh.box_outer : static_cast<long>(ntiles) * chunks;
  const int steps = sh.row_tiles ? n / (sh.box_inner * sh.loads) : chunk_rows / sh.box_outer;
  if (threadIdx.x == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (long t = blockIdx.x; t < tile_a; t += gridDim.x)
      for (int k = 0; k < steps; ++k) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect_tx(&full[st], stage_bytes);
        for (int j = 0; j < sh.loads; ++j) {
          if (sh.row_tiles)
            tma_load_2d(smem + st * stage_bytes + j * box_bytes, &tm, &full[st], (k * sh.loads + j) * sh.box_inner,
                        static_cast<int>(t * sh.box_outer));
          else
            tma_load_2d(smem + st * stage_bytes + j * box_bytes, &tm, &full[st],
                        static_cast<int>((t % ntiles) * sh.box_inner),
                        static_cast<int>((t / ntiles) * chunk_rows + k * sh.box_outer));
        }
        if (++st == stages) {
          st = 0;
          ph ^= 1;
        }
      }
  } else if (threadIdx.x == 32) {
    int st = 0;
    uint32_t ph = 0;
    for (long t = blockIdx.x; t < tile_a; t += gridDim.x)
      for (int k = 0; k < steps; ++k) {
        mbar_wait(&full[st], ph);
        mbar_arrive(&empty[st]);
        if (++st == stages) {
          st = 0;
          ph ^= 1;
        }
      }
  }
}

int main() {
  const int m = 1000000, n = 4096;
  float* x;
  cudaMalloc(&x, sizeof(float) * m * n);
  cudaMemset(x, 0, sizeof(float) * m * n);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  Shape shapes[] = {{"XW  {32,128} x1 sw128 (tf32 stage)", 32, 128, 1, true, true},
                    {"XW  {32,128} x2 sw128 (f16 stage)", 32, 128, 2, true, true},
                    {"XW  {32,128} x4 sw128", 32, 128, 4, true, true},
                    {"XW  {32,256} x2 sw128", 32, 256, 2, true, true},
                    {"XTU {128,32} (tf32 stage)", 128, 32, 1, false, false},
                    {"XTU {128,64} (f16 stage)", 128, 64, 1, false, false},
                    {"XTU {256,32}", 256, 32, 1, false, false}};
  int sms = 148;
  for (auto& sh : shapes) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(m)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(n) * 4};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(sh.box_inner), static_cast<cuuint32_t>(sh.box_outer)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sh.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("%s: encode failed %d\n", sh.name, r);
      continue;
    }
    const int stage_bytes = sh.box_inner * sh.box_outer * 4 * sh.loads;
    for (int stages : {4, 6}) {
      if (stages * stage_bytes > 200 * 1024) continue;
      const int smem = stages * stage_bytes + 2048;
      cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      stream<<<sms, 64, smem>>>(tm, m, n, sh, stages);
      cudaEventRecord(e0);
      for (int it = 0; it < 3; ++it) stream<<<sms, 64, smem>>>(tm, m, n, sh, stages);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 3;
      printf("%-40s stages %d (%3d KB): %.3f ms  %.0f GB/s  %s\n", sh.name, stages, stages * stage_bytes / 1024, ms,
             double(m) * n * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
