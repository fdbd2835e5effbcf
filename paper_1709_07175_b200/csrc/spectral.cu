// Device building blocks of the residual-norm metrics (proj/core/src/metrics.cpp:148-308,
// spectral_norm.cpp:23-57): matrix-vector products with X (dense row-major
// fp32/fp64 or CSR/CSC), tall-skinny products with an m x l basis, squared
// norms. Every reduction runs in a fixed order per launch (deterministic);
// the orders are the GPU's, not the reference's sequential ones.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lpca {

namespace {

constexpr int kRowWarps = 8;  // warps per CTA in the warp-per-row kernels

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y[i] = sum_j X[i][j] v[j], one warp per row (dense row-major, ld)
template <typename T>
__global__ void __launch_bounds__(32 * kRowWarps) matvec_dense_kernel(const T* __restrict__ x, index_t ld, index_t m,
                                                                      index_t n, const double* __restrict__ v,
                                                                      double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (index_t i = static_cast<index_t>(blockIdx.x) * kRowWarps + threadIdx.x / 32; i < m;
       i += static_cast<index_t>(gridDim.x) * kRowWarps) {
    const T* row = x + i * ld;
    double s = 0.0;
    for (index_t j = lane; j < n; j += 32) s = fma(static_cast<double>(row[j]), v[j], s);
    s = warp_sum_d(s);
    if (lane == 0) y[i] = s;
  }
}

// y[i] = sum_p val[p] v[col[p]] over row i's CSR entries, one warp per row
__global__ void __launch_bounds__(32 * kRowWarps) matvec_csr_kernel(const std::int64_t* __restrict__ rp,
                                                                    const std::int32_t* __restrict__ ci,
                                                                    const double* __restrict__ rv, index_t m,
                                                                    const double* __restrict__ v,
                                                                    double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (index_t i = static_cast<index_t>(blockIdx.x) * kRowWarps + threadIdx.x / 32; i < m;
       i += static_cast<index_t>(gridDim.x) * kRowWarps) {
    double s = 0.0;
    for (std::int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) s = fma(rv[p], v[ci[p]], s);
    s = warp_sum_d(s);
    if (lane == 0) y[i] = s;
  }
}

// part[c][j] = sum_{i in chunk c} X[i][j] t[i]: thread per column (coalesced
// along the row), rows of the chunk in order
template <typename T>
__global__ void __launch_bounds__(256) matvec_t_dense_kernel(const T* __restrict__ x, index_t ld, index_t m, index_t n,
                                                             const double* __restrict__ t, index_t chunk,
                                                             double* __restrict__ part) {
  const index_t j = static_cast<index_t>(blockIdx.x) * 256 + threadIdx.x;
  const index_t c = blockIdx.y;
  if (j >= n) return;
  const index_t i0 = c * chunk, i1 = i0 + chunk < m ? i0 + chunk : m;
  double s = 0.0;
  for (index_t i = i0; i < i1; ++i) s = fma(static_cast<double>(x[i * ld + j]), t[i], s);
  part[c * n + j] = s;
}

// y[j] = sum_p val[p] t[row[p]] over column j's CSC entries, one warp per column
__global__ void __launch_bounds__(32 * kRowWarps) matvec_t_csc_kernel(const std::int64_t* __restrict__ cp,
                                                                      const std::int32_t* __restrict__ ri,
                                                                      const double* __restrict__ cv, index_t n,
                                                                      const double* __restrict__ t,
                                                                      double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (index_t j = static_cast<index_t>(blockIdx.x) * kRowWarps + threadIdx.x / 32; j < n;
       j += static_cast<index_t>(gridDim.x) * kRowWarps) {
    double s = 0.0;
    for (std::int64_t p = cp[j] + lane; p < cp[j + 1]; p += 32) s = fma(cv[p], t[ri[p]], s);
    s = warp_sum_d(s);
    if (lane == 0) y[j] = s;
  }
}

// part[c][r] = sum_{i in chunk c} U[r*ldu + i] t[i]: warp per column r of the
// basis, lanes along the chunk's rows
__global__ void __launch_bounds__(32 * kRowWarps) basis_t_kernel(const double* __restrict__ u, index_t ldu, index_t m,
                                                                 index_t l, const double* __restrict__ t,
                                                                 index_t chunk, double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const index_t c = blockIdx.x;
  const index_t i0 = c * chunk, i1 = i0 + chunk < m ? i0 + chunk : m;
  for (index_t r = threadIdx.x / 32; r < l; r += kRowWarps) {
    const double* ur = u + r * ldu;
    double s = 0.0;
    for (index_t i = i0 + lane; i < i1; i += 32) s = fma(ur[i], t[i], s);
    s = warp_sum_d(s);
    if (lane == 0) part[c * l + r] = s;
  }
}

// y[i] = t[i] - sum_r U[r*ldu + i] s[r]
__global__ void basis_sub_kernel(const double* __restrict__ u, index_t ldu, index_t m, index_t l,
                                 const double* __restrict__ s, const double* __restrict__ t, double* __restrict__ y) {
  for (index_t i = static_cast<index_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<index_t>(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (index_t r = 0; r < l; ++r) acc = fma(u[r * ldu + i], s[r], acc);
    y[i] = t[i] - acc;
  }
}

// part[b] = sum of squares of this CTA's grid-stride share of the rows of a
// (rows x cols, ld) matrix of T
template <typename T>
__global__ void __launch_bounds__(256) sumsq_kernel(const T* __restrict__ a, index_t ld, index_t rows, index_t cols,
                                                    double* __restrict__ part) {
  __shared__ double red[8];
  double s = 0.0;
  const index_t count = rows * cols;
  for (index_t idx = static_cast<index_t>(blockIdx.x) * 256 + threadIdx.x; idx < count;
       idx += static_cast<index_t>(gridDim.x) * 256) {
    const index_t i = idx / cols, j = idx - i * cols;
    const double v = static_cast<double>(a[i * ld + j]);
    s = fma(v, v, s);
  }
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// s_out = Rinv (Rinv^T s) for Rinv = L^{-T} (upper, column-major l x l):
// (U^T U)^{-1} s through the Cholesky factor (Cholesky::solve_in_place,
// lazy_projector.cpp:52-68). One CTA.
__global__ void chol_solve_kernel(const double* __restrict__ rinv, index_t l, const double* __restrict__ s,
                                  double* __restrict__ tmp, double* __restrict__ out) {
  for (index_t i = threadIdx.x; i < l; i += blockDim.x) {  // tmp = Rinv^T s (lower)
    double acc = 0.0;
    for (index_t r = 0; r <= i; ++r) acc = fma(rinv[i * l + r], s[r], acc);
    tmp[i] = acc;
  }
  __syncthreads();
  for (index_t i = threadIdx.x; i < l; i += blockDim.x) {  // out = Rinv tmp (upper)
    double acc = 0.0;
    for (index_t r = i; r < l; ++r) acc = fma(rinv[r * l + i], tmp[r], acc);
    out[i] = acc;
  }
}

// dense row-major m x n (zeroed here) from CSR, one warp per row
__global__ void csr_to_dense_kernel(const std::int64_t* __restrict__ rp, const std::int32_t* __restrict__ ci,
                                    const double* __restrict__ rv, index_t m, index_t n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (index_t i = static_cast<index_t>(blockIdx.x) * kRowWarps + threadIdx.x / 32; i < m;
       i += static_cast<index_t>(gridDim.x) * kRowWarps) {
    double* row = out + i * n;
    for (index_t j = lane; j < n; j += 32) row[j] = 0.0;
    __syncwarp();
    for (std::int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) row[ci[p]] = rv[p];
  }
}

unsigned grid_for(index_t units, int per_cta) {
  index_t g = ceil_div(units, per_cta);
  if (g > 148 * 8) g = 148 * 8;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

}  // namespace

void launch_matvec(cudaStream_t s, int dtype, const void* x, index_t ld, index_t m, index_t n, const std::int64_t* rp,
                   const std::int32_t* ci, const double* rv, const double* v, double* y) {
  if (m <= 0) return;
  if (rp) {
    matvec_csr_kernel<<<grid_for(m, kRowWarps), 32 * kRowWarps, 0, s>>>(rp, ci, rv, m, v, y);
  } else if (dtype == 4) {
    matvec_dense_kernel<float><<<grid_for(m, kRowWarps), 32 * kRowWarps, 0, s>>>(static_cast<const float*>(x), ld, m,
                                                                                n, v, y);
  } else {
    matvec_dense_kernel<double><<<grid_for(m, kRowWarps), 32 * kRowWarps, 0, s>>>(static_cast<const double*>(x), ld,
                                                                                 m, n, v, y);
  }
}

index_t matvec_t_chunks(index_t m, index_t n) {
  const index_t col_ctas = ceil_div(n, 256);
  index_t chunks = ceil_div(148 * 8, col_ctas > 0 ? col_ctas : 1);
  const index_t max_chunks = ceil_div(m, 64);
  if (chunks > max_chunks) chunks = max_chunks;
  return chunks < 1 ? 1 : chunks;
}

void launch_matvec_t(cudaStream_t s, int dtype, const void* x, index_t ld, index_t m, index_t n,
                     const std::int64_t* cp, const std::int32_t* ri, const double* cv, const double* t, double* part,
                     double* y) {
  if (n <= 0) return;
  if (cp) {
    matvec_t_csc_kernel<<<grid_for(n, kRowWarps), 32 * kRowWarps, 0, s>>>(cp, ri, cv, n, t, y);
    return;
  }
  if (m <= 0) {
    launch_zero(s, y, sizeof(double) * n);
    return;
  }
  const index_t chunks = matvec_t_chunks(m, n);
  const index_t chunk = ceil_div(m, chunks);
  const dim3 grid(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(chunks));
  if (dtype == 4)
    matvec_t_dense_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), ld, m, n, t, chunk, part);
  else
    matvec_t_dense_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(x), ld, m, n, t, chunk, part);
  launch_reduce_partials(s, part, chunks, n, y);
}

index_t basis_t_chunks(index_t m) {
  index_t chunks = ceil_div(m, 4096);
  if (chunks > 148 * 4) chunks = 148 * 4;
  return chunks < 1 ? 1 : chunks;
}

void launch_basis_t(cudaStream_t s, const double* u, index_t ldu, index_t m, index_t l, const double* t,
                    double* part, double* out) {
  if (l <= 0) return;
  if (m <= 0) {
    launch_zero(s, out, sizeof(double) * l);
    return;
  }
  const index_t chunks = basis_t_chunks(m);
  basis_t_kernel<<<static_cast<unsigned>(chunks), 32 * kRowWarps, 0, s>>>(u, ldu, m, l, t, ceil_div(m, chunks), part);
  launch_reduce_partials(s, part, chunks, l, out);
}

void launch_basis_sub(cudaStream_t s, const double* u, index_t ldu, index_t m, index_t l, const double* sv,
                      const double* t, double* y) {
  if (m <= 0) return;
  basis_sub_kernel<<<grid_for(m, 256), 256, 0, s>>>(u, ldu, m, l, sv, t, y);
}

index_t sumsq_blocks(index_t count) {
  index_t g = ceil_div(count, 256 * 16);
  if (g > 148 * 4) g = 148 * 4;
  return g < 1 ? 1 : g;
}

void launch_sumsq(cudaStream_t s, int dtype, const void* a, index_t ld, index_t rows, index_t cols, double* part) {
  const index_t g = sumsq_blocks(rows * cols);
  if (rows * cols <= 0) {
    launch_zero(s, part, sizeof(double) * g);
    return;
  }
  if (dtype == 4)
    sumsq_kernel<float><<<static_cast<unsigned>(g), 256, 0, s>>>(static_cast<const float*>(a), ld, rows, cols, part);
  else
    sumsq_kernel<double><<<static_cast<unsigned>(g), 256, 0, s>>>(static_cast<const double*>(a), ld, rows, cols, part);
}

void launch_csr_to_dense(cudaStream_t s, index_t m, index_t n, const std::int64_t* rp, const std::int32_t* ci,
                         const double* rv, double* out) {
  if (m <= 0 || n <= 0) return;
  csr_to_dense_kernel<<<grid_for(m, kRowWarps), 32 * kRowWarps, 0, s>>>(rp, ci, rv, m, n, out);
}

void launch_chol_solve(cudaStream_t s, const double* rinv, index_t l, const double* sv, double* tmp, double* out) {
  if (l <= 0) return;
  chol_solve_kernel<<<1, 256, 0, s>>>(rinv, l, sv, tmp, out);
}

}  // namespace lpca
