// Sparse-X kernels (the reference's native input, SparseMatrix in canonical CSC:
// proj/core/src/kernels.cpp:30-113). X lives on the device twice — CSR for the
// row gathers of spmm (U = X W, Y = X V) and CSC for the column gathers of
// gemm_t (F = U^T X) — both with 32-bit indices and fp64 values.
//
// Accumulation order is the reference's: spmm sums each output U[i][c] over the
// row's nonzeros in ascending column order j (skipping W[j][c] == 0), and gemm_t
// sums F[c][j] over column j's nonzeros in ascending row order, each term as a
// separate multiply and add. The results are therefore bitwise equal to the
// reference's on the same inputs (the compiled reference uses -ffp-contract=off).
//
// Both are memory-latency bound gathers: one warp per output row (spmm) or
// column (gemm_t), lanes across the w (or l) outputs of that row/column, so
// the gathered W / U rows are read as coalesced, row-major, 8-byte vectors.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lpca {

namespace {

constexpr int kWarpsPerBlock = 8;

// U[i][c] (out at i * ors + c * ocs) = sum_{p in row i} v[p] * wt[col[p]][c],
// wt row-major n x w (ld ldw). kPer = outputs per lane (w <= 32 kPer).
template <int kPer, typename TO>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    spmm_csr_kernel(index_t m, const std::int64_t* __restrict__ row_ptr, const std::int32_t* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ wt, index_t ldw, int w,
                    TO* __restrict__ out, index_t ors, index_t ocs) {
  const int lane = threadIdx.x & 31;
  for (index_t i = blockIdx.x * static_cast<index_t>(kWarpsPerBlock) + threadIdx.x / 32; i < m;
       i += static_cast<index_t>(gridDim.x) * kWarpsPerBlock) {
    double acc[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) acc[t] = 0.0;
    const std::int64_t p1 = row_ptr[i + 1];
    for (std::int64_t p = row_ptr[i]; p < p1; ++p) {
      const double v = __ldg(val + p);
      const double* wr = wt + static_cast<index_t>(__ldg(col + p)) * ldw;
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const int c = lane + 32 * t;
        if (c < w) {
          const double b = __ldg(wr + c);
          if (b != 0.0) acc[t] = __dadd_rn(acc[t], __dmul_rn(v, b));
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int c = lane + 32 * t;
      if (c < w) out[i * ors + static_cast<index_t>(c) * ocs] = static_cast<TO>(acc[t]);
    }
  }
}

// F[c][j] (column-major l x n) (+)= sum_{p in column j} v[p] * u[row[p]][c],
// u row-major m x l (ld ldu).
template <int kPer>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    gemm_t_csc_kernel(index_t n, const std::int64_t* __restrict__ col_ptr, const std::int32_t* __restrict__ row,
                      const double* __restrict__ val, const double* __restrict__ u, index_t ldu, int l,
                      double* __restrict__ f, bool accumulate) {
  const int lane = threadIdx.x & 31;
  for (index_t j = blockIdx.x * static_cast<index_t>(kWarpsPerBlock) + threadIdx.x / 32; j < n;
       j += static_cast<index_t>(gridDim.x) * kWarpsPerBlock) {
    double* fc = f + j * l;
    double acc[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int c = lane + 32 * t;
      acc[t] = accumulate && c < l ? fc[c] : 0.0;
    }
    const std::int64_t p1 = col_ptr[j + 1];
    for (std::int64_t p = col_ptr[j]; p < p1; ++p) {
      const double v = __ldg(val + p);
      const double* ur = u + static_cast<index_t>(__ldg(row + p)) * ldu;
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const int c = lane + 32 * t;
        if (c < l) acc[t] = __dadd_rn(acc[t], __dmul_rn(v, __ldg(ur + c)));
      }
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int c = lane + 32 * t;
      if (c < l) fc[c] = acc[t];
    }
  }
}

unsigned grid_rows(index_t rows) {
  index_t g = ceil_div(rows, kWarpsPerBlock);
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

template <typename TO>
void spmm_dispatch(cudaStream_t s, index_t m, const std::int64_t* rp, const std::int32_t* ci, const double* v,
                   const double* wt, index_t ldw, index_t w, TO* out, index_t ors, index_t ocs) {
  const unsigned g = grid_rows(m);
  const int wi = static_cast<int>(w);
  if (w <= 32)
    spmm_csr_kernel<1, TO><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, rp, ci, v, wt, ldw, wi, out, ors, ocs);
  else if (w <= 64)
    spmm_csr_kernel<2, TO><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, rp, ci, v, wt, ldw, wi, out, ors, ocs);
  else if (w <= 128)
    spmm_csr_kernel<4, TO><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, rp, ci, v, wt, ldw, wi, out, ors, ocs);
  else if (w <= 256)
    spmm_csr_kernel<8, TO><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, rp, ci, v, wt, ldw, wi, out, ors, ocs);
  else if (w <= 512)
    spmm_csr_kernel<16, TO><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, rp, ci, v, wt, ldw, wi, out, ors, ocs);
  else
    throw Error(kInvalidArgument, "sparse spmm: at most 512 output columns per pass");
}

}  // namespace

void launch_spmm_csr(cudaStream_t s, index_t m, const std::int64_t* row_ptr, const std::int32_t* col,
                     const double* val, const double* wt, index_t ldw, index_t w, void* out, int out_dtype,
                     index_t ors, index_t ocs) {
  if (m <= 0 || w <= 0) return;
  for (index_t c0 = 0; c0 < w; c0 += 512) {  // wider W: 512-column slices
    const index_t wc = w - c0 < 512 ? w - c0 : 512;
    if (out_dtype == 4)
      spmm_dispatch<float>(s, m, row_ptr, col, val, wt + c0, ldw, wc, static_cast<float*>(out) + c0 * ocs, ors, ocs);
    else
      spmm_dispatch<double>(s, m, row_ptr, col, val, wt + c0, ldw, wc, static_cast<double*>(out) + c0 * ocs, ors,
                            ocs);
  }
}

void launch_gemm_t_csc(cudaStream_t s, index_t n, const std::int64_t* col_ptr, const std::int32_t* row,
                       const double* val, const double* u, index_t ldu, index_t l, double* f, bool accumulate) {
  if (n <= 0 || l <= 0) return;
  if (l > 512) throw Error(kInvalidArgument, "sparse gemm_t: at most 512 sketch columns");
  const unsigned g = grid_rows(n);
  const int li = static_cast<int>(l);
  if (l <= 32)
    gemm_t_csc_kernel<1><<<g, 32 * kWarpsPerBlock, 0, s>>>(n, col_ptr, row, val, u, ldu, li, f, accumulate);
  else if (l <= 64)
    gemm_t_csc_kernel<2><<<g, 32 * kWarpsPerBlock, 0, s>>>(n, col_ptr, row, val, u, ldu, li, f, accumulate);
  else if (l <= 128)
    gemm_t_csc_kernel<4><<<g, 32 * kWarpsPerBlock, 0, s>>>(n, col_ptr, row, val, u, ldu, li, f, accumulate);
  else if (l <= 256)
    gemm_t_csc_kernel<8><<<g, 32 * kWarpsPerBlock, 0, s>>>(n, col_ptr, row, val, u, ldu, li, f, accumulate);
  else
    gemm_t_csc_kernel<16><<<g, 32 * kWarpsPerBlock, 0, s>>>(n, col_ptr, row, val, u, ldu, li, f, accumulate);
}

}  // namespace lpca
