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

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

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
    // the row's (column, value) pairs 32 at a time, one per lane; kU nonzeros'
    // W rows loaded together, then added in ascending p (the reference's order)
    constexpr int kU = kPer <= 4 ? 4 : (kPer <= 8 ? 2 : 1);
    for (std::int64_t p0 = row_ptr[i]; p0 < p1; p0 += 32) {
      const int cnt = p1 - p0 < 32 ? static_cast<int>(p1 - p0) : 32;
      const int cj = lane < cnt ? __ldg(col + p0 + lane) : 0;
      const double cv = lane < cnt ? __ldg(val + p0 + lane) : 0.0;
      for (int q0 = 0; q0 < cnt; q0 += kU) {
        double v[kU], b[kU][kPer];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int src = q0 + u < cnt ? q0 + u : 0;
          v[u] = __shfl_sync(0xffffffffu, cv, src);
          const double* wr = wt + static_cast<index_t>(__shfl_sync(0xffffffffu, cj, src)) * ldw;
#pragma unroll
          for (int t = 0; t < kPer; ++t) {
            const int c = lane + 32 * t;
            b[u][t] = (q0 + u < cnt && c < w) ? __ldg(wr + c) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int t = 0; t < kPer; ++t)
            if (b[u][t] != 0.0) acc[t] = __dadd_rn(acc[t], __dmul_rn(v[u], b[u][t]));
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
    // as spmm_csr_kernel: (row, value) pairs 32 at a time, added in ascending p;
    // one U row at a time (U rarely fits L2: the gathers need occupancy more
    // than per-warp ILP — 4 rows in flight made F 1.8x slower, 2 rows 1.13x)
    constexpr int kU = 1;
    for (std::int64_t p0 = col_ptr[j]; p0 < p1; p0 += 32) {
      const int cnt = p1 - p0 < 32 ? static_cast<int>(p1 - p0) : 32;
      const int cr = lane < cnt ? __ldg(row + p0 + lane) : 0;
      const double cv = lane < cnt ? __ldg(val + p0 + lane) : 0.0;
      for (int q0 = 0; q0 < cnt; q0 += kU) {
        double v[kU], b[kU][kPer];
#pragma unroll
        for (int uu = 0; uu < kU; ++uu) {
          const int src = q0 + uu < cnt ? q0 + uu : 0;
          v[uu] = __shfl_sync(0xffffffffu, cv, src);
          const double* ur = u + static_cast<index_t>(__shfl_sync(0xffffffffu, cr, src)) * ldu;
#pragma unroll
          for (int t = 0; t < kPer; ++t) {
            const int c = lane + 32 * t;
            b[uu][t] = (q0 + uu < cnt && c < l) ? __ldg(ur + c) : 0.0;
          }
        }
#pragma unroll
        for (int uu = 0; uu < kU; ++uu)
          if (q0 + uu < cnt) {
#pragma unroll
            for (int t = 0; t < kPer; ++t)
              if (lane + 32 * t < l) acc[t] = __dadd_rn(acc[t], __dmul_rn(v[uu], b[uu][t]));
          }
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

// ---- sparse X times a {-1, 0, +1} W (the very sparse Omega, unscaled) -------------
// The dense-W gather reads W's whole row (8 l bytes) per nonzero of X, from L2
// (a 1.19G-nonzero X at l = 100: 0.95 TB of L2 reads per sketch). For a sign
// pattern each row of W is two bit masks, nonzero and negative, of
// wpad (multiple of 4) words: 32 B per row at l <= 128. The sums are the
// dense kernel's bit for bit: v * (+-1) is exactly +-v, and zero entries of W
// are skipped there too.
namespace {
__global__ void pm1_masks_kernel(const double* __restrict__ w, index_t n, int l, index_t ldw, int wpad,
                                 std::uint32_t* __restrict__ masks) {
  const index_t cells = n * wpad;
  for (index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; e < cells;
       e += static_cast<index_t>(gridDim.x) * blockDim.x) {
    const index_t j = e / wpad;
    const int t = static_cast<int>(e % wpad);
    std::uint32_t nz = 0, ng = 0;
    for (int b = 0; b < 32; ++b) {
      const int c = 32 * t + b;
      if (c >= l) break;
      const double v = w[static_cast<index_t>(c) * ldw + j];
      if (v != 0.0) nz |= 1u << b;
      if (v < 0.0) ng |= 1u << b;
    }
    masks[j * 2 * wpad + t] = nz;
    masks[j * 2 * wpad + wpad + t] = ng;
  }
}

template <int kPer, typename TO>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    spmm_csr_pm1_kernel(index_t m, const std::int64_t* __restrict__ row_ptr, const std::int32_t* __restrict__ col,
                        const double* __restrict__ val, const std::uint32_t* __restrict__ masks, int wpad, int w,
                        TO* __restrict__ out, index_t ors, index_t ocs) {
  const int lane = threadIdx.x & 31;
  for (index_t i = blockIdx.x * static_cast<index_t>(kWarpsPerBlock) + threadIdx.x / 32; i < m;
       i += static_cast<index_t>(gridDim.x) * kWarpsPerBlock) {
    double acc[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) acc[t] = 0.0;
    const std::int64_t p1 = row_ptr[i + 1];
    // (column, value) pairs 32 at a time, one per lane, then one nonzero at a
    // time in ascending p (the masks are one 32 B line; loading 4 nonzeros'
    // masks together measured slower: 82 -> 90 ms at 1.19G nonzeros)
    for (std::int64_t p0 = row_ptr[i]; p0 < p1; p0 += 32) {
      const int cnt = p1 - p0 < 32 ? static_cast<int>(p1 - p0) : 32;
      const int cj = lane < cnt ? __ldg(col + p0 + lane) : 0;
      const double cv = lane < cnt ? __ldg(val + p0 + lane) : 0.0;
      for (int q0 = 0; q0 < cnt; ++q0) {
        const double v = __shfl_sync(0xffffffffu, cv, q0);
        const uint4* mr =
            reinterpret_cast<const uint4*>(masks + static_cast<index_t>(__shfl_sync(0xffffffffu, cj, q0)) * 2 * wpad);
        std::uint32_t nz[kPer], ng[kPer];
#pragma unroll
        for (int q = 0; q < (kPer + 3) / 4; ++q) {
          const uint4 a = __ldg(mr + q), b = __ldg(mr + wpad / 4 + q);
          const std::uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (4 * q + r < kPer) {
              nz[4 * q + r] = av[r];
              ng[4 * q + r] = bv[r];
            }
        }
#pragma unroll
        for (int t = 0; t < kPer; ++t)
          if ((nz[t] >> lane) & 1u) acc[t] = __dadd_rn(acc[t], ((ng[t] >> lane) & 1u) ? -v : v);
      }
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int c = lane + 32 * t;
      if (c < w) out[i * ors + static_cast<index_t>(c) * ocs] = static_cast<TO>(acc[t]);
    }
  }
}
}  // namespace

int pm1_mask_words(index_t l) { return static_cast<int>(((l + 31) / 32 + 3) / 4 * 4); }

void launch_pm1_masks(cudaStream_t s, const double* w, index_t n, index_t l, index_t ldw, std::uint32_t* masks) {
  if (n <= 0) return;
  const int wpad = pm1_mask_words(l);
  pm1_masks_kernel<<<static_cast<unsigned>(ceil_div(n * wpad, 256) < 148 * 32 ? ceil_div(n * wpad, 256) : 148 * 32), 256, 0, s>>>(w, n, static_cast<int>(l), ldw, wpad, masks);
}

void launch_spmm_csr_pm1(cudaStream_t s, index_t m, const std::int64_t* row_ptr, const std::int32_t* col,
                         const double* val, const std::uint32_t* masks, index_t w, double* out, index_t ors,
                         index_t ocs) {
  if (m <= 0 || w <= 0) return;
  if (w > 512) throw Error(kInvalidArgument, "sparse spmm (sign W): at most 512 output columns");
  const unsigned g = grid_rows(m);
  const int wp = pm1_mask_words(w), wi = static_cast<int>(w);
  if (w <= 32)
    spmm_csr_pm1_kernel<1, double><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, row_ptr, col, val, masks, wp, wi, out, ors, ocs);
  else if (w <= 64)
    spmm_csr_pm1_kernel<2, double><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, row_ptr, col, val, masks, wp, wi, out, ors, ocs);
  else if (w <= 128)
    spmm_csr_pm1_kernel<4, double><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, row_ptr, col, val, masks, wp, wi, out, ors, ocs);
  else if (w <= 256)
    spmm_csr_pm1_kernel<8, double><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, row_ptr, col, val, masks, wp, wi, out, ors, ocs);
  else
    spmm_csr_pm1_kernel<16, double><<<g, 32 * kWarpsPerBlock, 0, s>>>(m, row_ptr, col, val, masks, wp, wi, out, ors, ocs);
}

// ---- CSC staging on the device (stage_x) ------------------------------------------
// A host CSC crosses PCIe as the caller holds it (int64 col_ptr / row_idx,
// fp32 or fp64 values); validation, the 32-bit row indices, fp64 values and
// the CSR copy are built here instead of by a serial host pass (a 1.2G-entry
// X took ~50 s on the host, most of it the CSR counting sort's scattered
// writes). Validation keeps the host loop's order: the first entry p (column
// major) failing any check, and for that entry the first check in the order
// range, strictly increasing, explicit zero, non-finite (first = 4 p + code).
namespace {
template <typename T>
__global__ void csc_check_kernel(index_t n, index_t rows, const std::int64_t* __restrict__ cp,
                                 const std::int64_t* __restrict__ ri64, const T* __restrict__ val,
                                 std::int32_t* __restrict__ ri, std::int32_t* __restrict__ colof,
                                 double* __restrict__ cv, unsigned long long* first) {
  const int lane = threadIdx.x & 31;
  for (index_t j = blockIdx.x * static_cast<index_t>(kWarpsPerBlock) + threadIdx.x / 32; j < n;
       j += static_cast<index_t>(gridDim.x) * kWarpsPerBlock) {
    const std::int64_t lo = cp[j], hi = cp[j + 1];
    for (std::int64_t p = lo + lane; p < hi; p += 32) {
      const std::int64_t r = ri64[p];
      const double v = static_cast<double>(val[p]);
      int code = -1;
      if (r < 0 || r >= rows) code = 0;
      else if (p > lo && r <= ri64[p - 1]) code = 1;
      else if (v == 0.0) code = 2;
      else if (!isfinite(v)) code = 3;
      if (code >= 0) atomicMin(first, static_cast<unsigned long long>(p) * 4ull + static_cast<unsigned>(code));
      ri[p] = static_cast<std::int32_t>(r);
      colof[p] = static_cast<std::int32_t>(j);
      cv[p] = v;
    }
  }
}

__global__ void row_count_kernel(index_t nnz, const std::int32_t* __restrict__ ri, std::int64_t* __restrict__ cnt) {
  for (index_t p = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; p < nnz;
       p += static_cast<index_t>(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + ri[p]), 1ull);
}

unsigned grid_flat(index_t count) {
  index_t g = ceil_div(count, 256);
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

int row_bits(index_t m) {
  int b = 1;
  while (b < 31 && (index_t(1) << b) < m) ++b;
  return b;
}
}  // namespace

std::size_t csc_stage_temp_bytes(index_t m, index_t nnz) {
  std::size_t sort_i = 0, sort_d = 0, scan_b = 0;
  const int n32 = static_cast<int>(nnz);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_i, static_cast<const std::int32_t*>(nullptr),
                                  static_cast<std::int32_t*>(nullptr), static_cast<const std::int32_t*>(nullptr),
                                  static_cast<std::int32_t*>(nullptr), n32, 0, row_bits(m));
  cub::DeviceRadixSort::SortPairs(nullptr, sort_d, static_cast<const std::int32_t*>(nullptr),
                                  static_cast<std::int32_t*>(nullptr), static_cast<const double*>(nullptr),
                                  static_cast<double*>(nullptr), n32, 0, row_bits(m));
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, static_cast<std::int64_t*>(nullptr),
                                static_cast<std::int64_t*>(nullptr), static_cast<int>(m + 1));
  std::size_t b = sort_i > sort_d ? sort_i : sort_d;
  return b > scan_b ? b : scan_b;
}

void launch_csc_check(cudaStream_t s, index_t n, index_t rows, const std::int64_t* cp, const std::int64_t* ri64,
                      const void* val, int dtype, std::int32_t* ri, std::int32_t* colof, double* cv,
                      unsigned long long* first) {
  if (n <= 0) return;
  LPCA_CUDA(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), s));
  const unsigned g = grid_rows(n);
  if (dtype == 4)
    csc_check_kernel<float><<<g, 32 * kWarpsPerBlock, 0, s>>>(n, rows, cp, ri64, static_cast<const float*>(val), ri,
                                                              colof, cv, first);
  else
    csc_check_kernel<double><<<g, 32 * kWarpsPerBlock, 0, s>>>(n, rows, cp, ri64, static_cast<const double*>(val),
                                                               ri, colof, cv, first);
}

// CSR from the checked CSC: stable radix sorts of the entries by row keep each
// row's columns ascending (the reference's accumulation order, as the host
// counting sort did) — one carrying the columns straight into ci, one the
// values into rv (two sorts instead of a sorted permutation and a random
// gather: 21 + 55 ms -> ~40 ms at 1.19G entries); row offsets by a histogram
// and an exclusive scan. cnt: m + 1 int64; keys_out: nnz int32; temp:
// csc_stage_temp_bytes.
void launch_csr_from_csc(cudaStream_t s, index_t m, index_t nnz, const std::int32_t* ri, const std::int32_t* colof,
                         const double* cv, std::int64_t* rp, std::int32_t* ci, double* rv, std::int64_t* cnt,
                         std::int32_t* keys_out, void* temp, std::size_t temp_bytes) {
  LPCA_CUDA(cudaMemsetAsync(cnt, 0, sizeof(std::int64_t) * static_cast<std::size_t>(m + 1), s));
  if (nnz > 0) row_count_kernel<<<grid_flat(nnz), 256, 0, s>>>(nnz, ri, cnt);
  std::size_t tb = temp_bytes;
  LPCA_CUDA(cub::DeviceScan::ExclusiveSum(temp, tb, cnt, rp, static_cast<int>(m + 1), s));
  if (nnz <= 0) return;
  tb = temp_bytes;
  LPCA_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, ri, keys_out, colof, ci, static_cast<int>(nnz), 0,
                                            row_bits(m), s));
  tb = temp_bytes;
  LPCA_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, ri, keys_out, cv, rv, static_cast<int>(nnz), 0,
                                            row_bits(m), s));
}

}  // namespace lpca
