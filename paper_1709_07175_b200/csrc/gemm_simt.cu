// SIMT tall-skinny GEMMs (FFMA for fp32 data, DFMA for fp64 data).
//
// These are the exact-order / fp64 path and the A/B baseline for the tcgen05
// split-TF32 kernels in gemm_tc.cu. Accumulation order is a fixed function of
// the shapes (CTA tiles own disjoint outputs; K is walked in ascending order),
// so results are bitwise reproducible run to run — the reference's determinism
// contract (proj/core/include/lazypca/kernels.hpp:5-9). In `exact` mode the fp64
// kernels use separate multiply and add in the reference's summation order,
// which reproduces the reference's spmm / gemm_t bit for bit on dense input.
#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.cuh"

namespace lpca {

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kThreads = 256;
constexpr int kFlushK = 256;  // fp32 partial sums span at most this many products

template <typename T, bool kExact>
struct Acc;

template <bool kExact>
struct Acc<double, kExact> {
  double v[4][4];
  __device__ void zero() {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) v[a][b] = 0.0;
  }
  __device__ __forceinline__ void add(int a, int b, double x, double y) {
    if constexpr (kExact)
      v[a][b] = __dadd_rn(v[a][b], __dmul_rn(x, y));
    else
      v[a][b] = fma(x, y, v[a][b]);
  }
  __device__ __forceinline__ void flush() {}
  __device__ __forceinline__ double get(int a, int b) const { return v[a][b]; }
};

template <bool kExact>
struct Acc<float, kExact> {
  float f[4][4];
  double d[4][4];
  __device__ void zero() {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        f[a][b] = 0.f;
        d[a][b] = 0.0;
      }
  }
  __device__ __forceinline__ void add(int a, int b, float x, float y) { f[a][b] = fmaf(x, y, f[a][b]); }
  __device__ __forceinline__ void flush() {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        d[a][b] += static_cast<double>(f[a][b]);
        f[a][b] = 0.f;
      }
  }
  __device__ __forceinline__ double get(int a, int b) const { return d[a][b]; }
};

// out[i*ors + c*ocs] = sum_j X[i, j] W[c, j]; CTA tile 64 rows x 64 columns.
template <typename T, typename TO, bool kExact>
__global__ void __launch_bounds__(kThreads) xw_simt_kernel(const T* __restrict__ x, index_t m,
                                                           index_t n, index_t ldx,
                                                           const T* __restrict__ w, index_t wc,
                                                           index_t ldw, TO* __restrict__ out,
                                                           index_t ors, index_t ocs) {
  __shared__ T As[kBK][kBM + 1];
  __shared__ T Bs[kBK][kBN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const index_t i0 = static_cast<index_t>(blockIdx.x) * kBM;
  const index_t c0 = static_cast<index_t>(blockIdx.y) * kBN;
  Acc<T, kExact> acc;
  acc.zero();
  int since_flush = 0;
  for (index_t k0 = 0; k0 < n; k0 += kBK) {
    for (int e = threadIdx.x; e < kBM * kBK; e += kThreads) {
      const int r = e / kBK, kk = e % kBK;
      const index_t gi = i0 + r, gk = k0 + kk;
      As[kk][r] = (gi < m && gk < n) ? x[gi * ldx + gk] : T(0);
    }
    for (int e = threadIdx.x; e < kBN * kBK; e += kThreads) {
      const int c = e / kBK, kk = e % kBK;
      const index_t gc = c0 + c, gk = k0 + kk;
      Bs[kk][c] = (gc < wc && gk < n) ? w[gc * ldw + gk] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      T av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc.add(a, b, av[a], bv[b]);
    }
    since_flush += kBK;
    if (since_flush >= kFlushK) {
      acc.flush();
      since_flush = 0;
    }
    __syncthreads();
  }
  acc.flush();
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const index_t gi = i0 + ty + 16 * a;
    if (gi >= m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const index_t gc = c0 + tx + 16 * b;
      if (gc < wc) out[gi * ors + gc * ocs] = static_cast<TO>(acc.get(a, b));
    }
  }
}

// part[c][j*l + r] = sum_{i in chunk c} U[i, r] X[i, j]; CTA tile 64 (r) x 64 (j).
template <typename T, bool kExact>
__global__ void __launch_bounds__(kThreads) utx_simt_kernel(const T* __restrict__ u, index_t ldu,
                                                            const T* __restrict__ x, index_t ldx,
                                                            index_t m, index_t l, index_t n,
                                                            index_t chunk_rows,
                                                            double* __restrict__ part) {
  __shared__ T Us[kBK][kBM + 1];
  __shared__ T Xs[kBK][kBN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const index_t j0 = static_cast<index_t>(blockIdx.x) * kBN;
  const index_t r0 = static_cast<index_t>(blockIdx.y) * kBM;
  const index_t chunk = blockIdx.z;
  const index_t row_begin = chunk * chunk_rows;
  const index_t row_end = row_begin + chunk_rows < m ? row_begin + chunk_rows : m;
  Acc<T, kExact> acc;
  acc.zero();
  int since_flush = 0;
  for (index_t i0 = row_begin; i0 < row_end; i0 += kBK) {
    for (int e = threadIdx.x; e < kBM * kBK; e += kThreads) {
      const int kk = e / kBM, rr = e % kBM;
      const index_t gi = i0 + kk, gr = r0 + rr;
      Us[kk][rr] = (gi < row_end && gr < l) ? u[gi * ldu + gr] : T(0);
    }
    for (int e = threadIdx.x; e < kBN * kBK; e += kThreads) {
      const int kk = e / kBN, jj = e % kBN;
      const index_t gi = i0 + kk, gj = j0 + jj;
      Xs[kk][jj] = (gi < row_end && gj < n) ? x[gi * ldx + gj] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      T uv[4], xv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) uv[a] = Us[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) xv[b] = Xs[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc.add(a, b, xv[b], uv[a]);
    }
    since_flush += kBK;
    if (since_flush >= kFlushK) {
      acc.flush();
      since_flush = 0;
    }
    __syncthreads();
  }
  acc.flush();
  double* dst = part + chunk * l * n;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const index_t gr = r0 + ty + 16 * a;
    if (gr >= l) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const index_t gj = j0 + tx + 16 * b;
      if (gj < n) dst[gj * l + gr] = acc.get(a, b);
    }
  }
}

__global__ void reduce_partials_kernel(const double* __restrict__ part, index_t nparts,
                                       index_t count, double* __restrict__ out) {
  for (index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<index_t>(gridDim.x) * blockDim.x) {
    double s = part[e];
    for (index_t c = 1; c < nparts; ++c) s += part[c * count + e];
    out[e] = s;
  }
}

// ---- fp64, free summation order: 128 x 128 CTA tiles on the fp64 tensor cores
// (DMMA m8n8k4), the next K slab prefetched into registers while the current
// one is multiplied. Used for the fp64 passes when the reference's exact order
// is not requested (c5).
constexpr int kFT = 128, kFK = 16;

// A slab [kFK][kFT] and B slab [kFK][kFT] in shared memory (padded rows).
struct F64Slabs {
  double a[kFK][kFT + 1];
  double b[kFK][kFT + 1];
};

// The 128 x 128 tile on the fp64 tensor cores (mma.sync m8n8k4 f64): warp w
// owns rows 64 (w / 4) .. +64 and columns 32 (w % 4) .. +32 as 8 x 4 tiles of
// 8 x 8; per K = 4 step a thread loads 8 A and 4 B values for 32 MMAs.
// Fragments: A[g][t], B[t][g], C[g][2t + {0,1}] with g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void f64_tile_mma(const F64Slabs& sm, int warp, int lane, double (&acc)[8][4][2]) {
  const int g = lane >> 2, t = lane & 3;
  const int rbase = 64 * (warp >> 2) + g, cbase = 32 * (warp & 3) + g;
#pragma unroll
  for (int k = 0; k < kFK; k += 4) {
    double av[8], bv[4];
#pragma unroll
    for (int rb = 0; rb < 8; ++rb) av[rb] = sm.a[k + t][rbase + 8 * rb];
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) bv[cb] = sm.b[k + t][cbase + 8 * cb];
#pragma unroll
    for (int rb = 0; rb < 8; ++rb)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) dmma_8x8x4(acc[rb][cb], av[rb], bv[cb]);
  }
}

// out[i*ors + c*ocs] = sum_k X[i, k] W[c, k] (X row-major ldx, W as w[c*ldw + k]).
template <typename TO>
__global__ void __launch_bounds__(256, 1) xw_f64_fast_kernel(const double* __restrict__ x, index_t m, index_t n,
                                                             index_t ldx, const double* __restrict__ w, index_t wc,
                                                             index_t ldw, TO* __restrict__ out, index_t ors,
                                                             index_t ocs) {
  extern __shared__ double f64_smem[];
  F64Slabs& sm = *reinterpret_cast<F64Slabs*>(f64_smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const index_t i0 = static_cast<index_t>(blockIdx.x) * kFT, c0 = static_cast<index_t>(blockIdx.y) * kFT;
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double ra[8], rb[8];  // this thread's share of the next slab: rows/cols e / 16, k e % 16
  auto fetch = [&](index_t k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + 256 * q, r = e / kFK, kk = e % kFK;
      const index_t gk = k0 + kk, gi = i0 + r, gc = c0 + r;
      ra[q] = (gi < m && gk < n) ? x[gi * ldx + gk] : 0.0;
      rb[q] = (gc < wc && gk < n) ? w[gc * ldw + gk] : 0.0;
    }
  };
  fetch(0);
  for (index_t k0 = 0; k0 < n; k0 += kFK) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + 256 * q, r = e / kFK, kk = e % kFK;
      sm.a[kk][r] = ra[q];
      sm.b[kk][r] = rb[q];
    }
    __syncthreads();
    if (k0 + kFK < n) fetch(k0 + kFK);  // in flight while this slab is multiplied
    f64_tile_mma(sm, warp, lane, acc);
    __syncthreads();
  }
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int rb = 0; rb < 8; ++rb) {
    const index_t gi = i0 + 64 * (warp >> 2) + 8 * rb + g;
    if (gi >= m) continue;
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const index_t gc = c0 + 32 * (warp & 3) + 8 * cb + 2 * t + h;
        if (gc < wc) out[gi * ors + gc * ocs] = static_cast<TO>(acc[rb][cb][h]);
      }
  }
}

// part[c][j*l + r] = sum_{i in chunk c} U[i, r] X[i, j] (U ldu, X ldx row-major).
__global__ void __launch_bounds__(256, 1) utx_f64_fast_kernel(const double* __restrict__ u, index_t ldu,
                                                              const double* __restrict__ x, index_t ldx, index_t m,
                                                              index_t l, index_t n, index_t chunk_rows,
                                                              double* __restrict__ part) {
  extern __shared__ double f64_smem[];
  F64Slabs& sm = *reinterpret_cast<F64Slabs*>(f64_smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const index_t j0 = static_cast<index_t>(blockIdx.x) * kFT, r0 = static_cast<index_t>(blockIdx.y) * kFT;
  const index_t chunk = blockIdx.z;
  const index_t row_begin = chunk * chunk_rows, row_end = row_begin + chunk_rows < m ? row_begin + chunk_rows : m;
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double ra[8], rb[8];  // slab element e: row kk = e / 128, column e % 128
  auto fetch = [&](index_t i0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + 256 * q, kk = e / kFT, c = e % kFT;
      const index_t gi = i0 + kk;
      const bool in = gi < row_end;
      ra[q] = (in && r0 + c < l) ? u[gi * ldu + r0 + c] : 0.0;
      rb[q] = (in && j0 + c < n) ? x[gi * ldx + j0 + c] : 0.0;
    }
  };
  fetch(row_begin);
  for (index_t i0 = row_begin; i0 < row_end; i0 += kFK) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + 256 * q, kk = e / kFT, c = e % kFT;
      sm.a[kk][c] = ra[q];
      sm.b[kk][c] = rb[q];
    }
    __syncthreads();
    if (i0 + kFK < row_end) fetch(i0 + kFK);
    f64_tile_mma(sm, warp, lane, acc);
    __syncthreads();
  }
  double* dst = part + chunk * l * n;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int rb = 0; rb < 8; ++rb) {
    const index_t r = r0 + 64 * (warp >> 2) + 8 * rb + g;
    if (r >= l) continue;
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const index_t j = j0 + 32 * (warp & 3) + 8 * cb + 2 * t + h;
        if (j < n) dst[j * l + r] = acc[rb][cb][h];
      }
  }
}

}  // namespace

template <typename T, typename TO>
void launch_xw_simt(cudaStream_t s, const T* x, index_t m, index_t n, index_t ldx, const T* w,
                    index_t wc, index_t ldw, TO* out, index_t ors, index_t ocs, bool exact) {
  if (m <= 0 || wc <= 0) return;
  if constexpr (std::is_same<T, double>::value) {
    if (!exact && wc > 64) {
      const dim3 g(static_cast<unsigned>(ceil_div(m, kFT)), static_cast<unsigned>(ceil_div(wc, kFT)));
      const int smem = static_cast<int>(sizeof(F64Slabs));
      LPCA_CUDA(cudaFuncSetAttribute(xw_f64_fast_kernel<TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      xw_f64_fast_kernel<TO><<<g, 256, smem, s>>>(x, m, n, ldx, w, wc, ldw, out, ors, ocs);
      return;
    }
  }
  dim3 grid(static_cast<unsigned>(ceil_div(m, kBM)), static_cast<unsigned>(ceil_div(wc, kBN)));
  if (exact)
    xw_simt_kernel<T, TO, true><<<grid, kThreads, 0, s>>>(x, m, n, ldx, w, wc, ldw, out, ors, ocs);
  else
    xw_simt_kernel<T, TO, false><<<grid, kThreads, 0, s>>>(x, m, n, ldx, w, wc, ldw, out, ors, ocs);
}

template <typename T>
void launch_utx_simt(cudaStream_t s, const T* u, index_t ldu, const T* x, index_t ldx, index_t m,
                     index_t l, index_t n, index_t chunk_rows, double* part, bool exact) {
  const index_t chunks = ceil_div(m, chunk_rows);
  if constexpr (std::is_same<T, double>::value) {
    if (!exact && l > 64 && n > 64) {
      const dim3 g(static_cast<unsigned>(ceil_div(n, kFT)), static_cast<unsigned>(ceil_div(l, kFT)),
                   static_cast<unsigned>(chunks));
      const int smem = static_cast<int>(sizeof(F64Slabs));
      LPCA_CUDA(cudaFuncSetAttribute(utx_f64_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      utx_f64_fast_kernel<<<g, 256, smem, s>>>(u, ldu, x, ldx, m, l, n, chunk_rows, part);
      return;
    }
  }
  dim3 grid(static_cast<unsigned>(ceil_div(n, kBN)), static_cast<unsigned>(ceil_div(l, kBM)),
            static_cast<unsigned>(chunks));
  if (exact)
    utx_simt_kernel<T, true><<<grid, kThreads, 0, s>>>(u, ldu, x, ldx, m, l, n, chunk_rows, part);
  else
    utx_simt_kernel<T, false><<<grid, kThreads, 0, s>>>(u, ldu, x, ldx, m, l, n, chunk_rows, part);
}

template <typename T>
void launch_syrk_partials(cudaStream_t s, const T* u, index_t ldu, index_t m, index_t l,
                          index_t chunk_rows, double* part) {
  launch_utx_simt<T>(s, u, ldu, u, ldu, m, l, l, chunk_rows, part, false);
}

namespace {
__global__ void add_f64_kernel(const double* __restrict__ x, double* __restrict__ y, index_t count) {
  for (index_t i = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<index_t>(gridDim.x) * blockDim.x)
    y[i] += x[i];
}
}  // namespace

void launch_add_f64(cudaStream_t s, const double* x, double* y, index_t count) {
  if (count <= 0) return;
  index_t g = ceil_div(count, 256);
  if (g > 148 * 8) g = 148 * 8;
  add_f64_kernel<<<static_cast<unsigned>(g), 256, 0, s>>>(x, y, count);
}

void launch_reduce_partials(cudaStream_t s, const double* part, index_t nparts, index_t count,
                            double* out) {
  index_t g = ceil_div(count, 256);
  if (g > 148 * 8) g = 148 * 8;
  reduce_partials_kernel<<<static_cast<unsigned>(g), 256, 0, s>>>(part, nparts, count, out);
}

template void launch_xw_simt<float, float>(cudaStream_t, const float*, index_t, index_t, index_t,
                                           const float*, index_t, index_t, float*, index_t, index_t, bool);
template void launch_xw_simt<float, double>(cudaStream_t, const float*, index_t, index_t, index_t,
                                            const float*, index_t, index_t, double*, index_t, index_t, bool);
template void launch_xw_simt<double, double>(cudaStream_t, const double*, index_t, index_t, index_t,
                                             const double*, index_t, index_t, double*, index_t, index_t, bool);
template void launch_xw_simt<double, float>(cudaStream_t, const double*, index_t, index_t, index_t,
                                            const double*, index_t, index_t, float*, index_t, index_t, bool);
template void launch_utx_simt<float>(cudaStream_t, const float*, index_t, const float*, index_t,
                                     index_t, index_t, index_t, index_t, double*, bool);
template void launch_utx_simt<double>(cudaStream_t, const double*, index_t, const double*, index_t,
                                      index_t, index_t, index_t, index_t, double*, bool);
template void launch_syrk_partials<float>(cudaStream_t, const float*, index_t, index_t, index_t,
                                          index_t, double*);
template void launch_syrk_partials<double>(cudaStream_t, const double*, index_t, index_t, index_t,
                                           index_t, double*);

}  // namespace lpca
