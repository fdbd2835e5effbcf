// Verification metrics at scale on the device (proj/core/src/metrics.cpp):
// chordal distance between two orthonormal bases in the cancellation-free
// residual form (:123-136) and the sampled pairwise distances of
// distance_preservation (:311-352). fp64 throughout; sums run in a fixed
// order per launch (deterministic), not the reference's sequential order.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lpca {

namespace {

// C (ka x kb, column-major) = A^T B for column-major A (n x ka), B (n x kb):
// 32 x 32 output tile per CTA, the n-sum staged through shared memory.
__global__ void __launch_bounds__(256) atb_kernel(const double* __restrict__ a, index_t n, index_t ka,
                                                  const double* __restrict__ b, index_t kb, double* __restrict__ c) {
  __shared__ double as[32][33];
  __shared__ double bs[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const index_t c0 = static_cast<index_t>(blockIdx.x) * 32, r0 = static_cast<index_t>(blockIdx.y) * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (index_t i0 = 0; i0 < n; i0 += 32) {
    for (int t = ty; t < 32; t += 8) {
      const index_t i = i0 + tx;
      as[t][tx] = (r0 + t < ka && i < n) ? a[(r0 + t) * n + i] : 0.0;  // as[r][i]
      bs[t][tx] = (c0 + t < kb && i < n) ? b[(c0 + t) * n + i] : 0.0;  // bs[c][i]
    }
    __syncthreads();
#pragma unroll 8
    for (int ii = 0; ii < 32; ++ii) {
      const double bv = bs[tx][ii];
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[t] = fma(as[ty + 8 * t][ii], bv, acc[t]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const index_t r = r0 + ty + 8 * t, col = c0 + tx;
    if (r < ka && col < kb) c[col * ka + r] = acc[t];
  }
}

// part[block] = sum over this CTA's tile of (A - B C)^2, A n x ka, B n x kb,
// C kb x ka (all column-major); tile 32 rows x 32 columns of A.
__global__ void __launch_bounds__(256) residual_sq_kernel(const double* __restrict__ a, index_t n, index_t ka,
                                                          const double* __restrict__ b, index_t kb,
                                                          const double* __restrict__ c, double* __restrict__ part) {
  __shared__ double bs[32][33];
  __shared__ double cs[32][33];
  __shared__ double red[8];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const index_t i0 = static_cast<index_t>(blockIdx.x) * 32, c0 = static_cast<index_t>(blockIdx.y) * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // (B C)[i0 + tx][c0 + ty + 8t]
  for (index_t r0 = 0; r0 < kb; r0 += 32) {
    for (int t = ty; t < 32; t += 8) {
      bs[t][tx] = (i0 + tx < n && r0 + t < kb) ? b[(r0 + t) * n + i0 + tx] : 0.0;     // bs[r][i]
      cs[t][tx] = (r0 + tx < kb && c0 + t < ka) ? c[(c0 + t) * kb + r0 + tx] : 0.0;  // cs[col][r]
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const double bv = bs[rr][tx];
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[t] = fma(bv, cs[ty + 8 * t][rr], acc[t]);
    }
    __syncthreads();
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const index_t i = i0 + tx, col = c0 + ty + 8 * t;
    if (i < n && col < ka) {
      const double d = a[col * n + i] - acc[t];
      s = fma(d, d, s);
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (tx == 0) red[ty] = s;
  __syncthreads();
  if (ty == 0 && tx == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// One warp per pair: ||x_i - x_j|| (dense row-major fp32/fp64 or CSR) and the
// reduced distances of row-major Y_a, Y_b (m x k, fp64; yb nullable).
template <typename T>
__global__ void pair_dense_kernel(const T* __restrict__ x, index_t ld, index_t n, const std::int64_t* __restrict__ pi,
                                  const std::int64_t* __restrict__ pj, index_t pairs, double* __restrict__ orig) {
  const int lane = threadIdx.x & 31;
  for (index_t p = blockIdx.x * static_cast<index_t>(blockDim.x / 32) + threadIdx.x / 32; p < pairs;
       p += static_cast<index_t>(gridDim.x) * (blockDim.x / 32)) {
    const T* a = x + pi[p] * ld;
    const T* b = x + pj[p] * ld;
    double s = 0.0;
    for (index_t c = lane; c < n; c += 32) {
      const double d = static_cast<double>(a[c]) - static_cast<double>(b[c]);
      s = fma(d, d, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) orig[p] = sqrt(s);
  }
}

__global__ void pair_csr_kernel(const std::int64_t* __restrict__ rp, const std::int32_t* __restrict__ ci,
                                const double* __restrict__ rv, const std::int64_t* __restrict__ pi,
                                const std::int64_t* __restrict__ pj, index_t pairs, double* __restrict__ orig) {
  // one thread per pair: a merge of the two sorted rows (sparse_row_distance, metrics.cpp:69-91)
  const index_t p = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x;
  if (p >= pairs) return;
  std::int64_t a = rp[pi[p]], ae = rp[pi[p] + 1], b = rp[pj[p]], be = rp[pj[p] + 1];
  double s = 0.0;
  while (a < ae || b < be) {
    double d;
    if (b >= be || (a < ae && ci[a] < ci[b])) {
      d = rv[a++];
    } else if (a >= ae || ci[b] < ci[a]) {
      d = -rv[b++];
    } else {
      d = rv[a++] - rv[b++];
    }
    s += d * d;
  }
  orig[p] = sqrt(s);
}

__global__ void pair_reduced_kernel(const double* __restrict__ ya, const double* __restrict__ yb, index_t k,
                                    const std::int64_t* __restrict__ pi, const std::int64_t* __restrict__ pj,
                                    index_t pairs, double* __restrict__ da, double* __restrict__ db) {
  const int lane = threadIdx.x & 31;
  for (index_t p = blockIdx.x * static_cast<index_t>(blockDim.x / 32) + threadIdx.x / 32; p < pairs;
       p += static_cast<index_t>(gridDim.x) * (blockDim.x / 32)) {
    double sa = 0.0, sb = 0.0;
    for (index_t c = lane; c < k; c += 32) {
      const double d = ya[pi[p] * k + c] - ya[pj[p] * k + c];
      sa = fma(d, d, sa);
      if (yb) {
        const double e = yb[pi[p] * k + c] - yb[pj[p] * k + c];
        sb = fma(e, e, sb);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
      da[p] = sqrt(sa);
      if (yb) db[p] = sqrt(sb);
    }
  }
}

unsigned pair_grid(index_t pairs) {
  index_t g = ceil_div(pairs, 8);
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

}  // namespace

void launch_atb(cudaStream_t s, const double* a, index_t n, index_t ka, const double* b, index_t kb, double* c) {
  if (ka <= 0 || kb <= 0) return;
  const dim3 grid(static_cast<unsigned>(ceil_div(kb, 32)), static_cast<unsigned>(ceil_div(ka, 32)));
  atb_kernel<<<grid, dim3(32, 8), 0, s>>>(a, n, ka, b, kb, c);
}

index_t residual_sq_blocks(index_t n, index_t ka) { return ceil_div(n, 32) * ceil_div(ka, 32); }

void launch_residual_sq(cudaStream_t s, const double* a, index_t n, index_t ka, const double* b, index_t kb,
                        const double* c, double* part) {
  if (n <= 0 || ka <= 0) return;
  const dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(ka, 32)));
  residual_sq_kernel<<<grid, dim3(32, 8), 0, s>>>(a, n, ka, b, kb, c, part);
}

void launch_pair_distances(cudaStream_t s, int dtype, const void* x, index_t ld, index_t n, const std::int64_t* rp,
                           const std::int32_t* ci, const double* rv, const double* ya, const double* yb, index_t k,
                           const std::int64_t* pi, const std::int64_t* pj, index_t pairs, double* orig, double* da,
                           double* db) {
  if (pairs <= 0) return;
  if (rp)
    pair_csr_kernel<<<static_cast<unsigned>(ceil_div(pairs, 128)), 128, 0, s>>>(rp, ci, rv, pi, pj, pairs, orig);
  else if (dtype == 4)
    pair_dense_kernel<float><<<pair_grid(pairs), 256, 0, s>>>(static_cast<const float*>(x), ld, n, pi, pj, pairs, orig);
  else
    pair_dense_kernel<double><<<pair_grid(pairs), 256, 0, s>>>(static_cast<const double*>(x), ld, n, pi, pj, pairs,
                                                                orig);
  pair_reduced_kernel<<<pair_grid(pairs), 256, 0, s>>>(ya, yb, k, pi, pj, pairs, da, db);
}

}  // namespace lpca
