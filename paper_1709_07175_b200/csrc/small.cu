// The l x l step on the device, fp64 throughout:
//   G = F F^T (dense_aat), symmetric eigendecomposition (parallel cyclic
//   Jacobi in one CTA), V = F^T U~ diag(sigma)^-1 with canonical signs
//   (truncated_svd_via_gram), and the Cholesky pieces of CholeskyQR2.
// Reference: proj/core/src/kernels.cpp:148-172, proj/core/src/jacobi.cpp:18-135,
// proj/core/src/truncated_svd.cpp:13-82, proj/core/src/lazy_projector.cpp:12-37.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lpca {

namespace {

// dense_aat: G(r, c) = sum_j F(c, j) * F(r, j), j ascending, separate multiply
// and add — the reference's exact rounding sequence, so G is bitwise equal to
// the reference's for equal F and bitwise symmetric by construction.
__global__ void gram_kernel(const double* __restrict__ f, index_t l, index_t n,
                            double* __restrict__ g) {
  const index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x;
  if (e >= l * l) return;
  const index_t c = e / l, r = e % l;
  double acc = 0.0;
  for (index_t j = 0; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(f[j * l + c], f[j * l + r]));
  g[c * l + r] = acc;
}

constexpr int kJacobiThreads = 1024;
constexpr int kMaxSweeps = 50;  // jacobi.cpp:64

__device__ __forceinline__ void block_max_reduce(double& v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < static_cast<int>(blockDim.x / 32) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
}

__device__ __forceinline__ void block_sum_reduce(double& v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < static_cast<int>(blockDim.x / 32) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
}

// Parallel cyclic Jacobi. Each round of the reference's round-robin schedule
// (jacobi.cpp:18-33) is a set of l/2 disjoint pairs; rotations on disjoint
// pairs commute and their angles depend only on their own 2x2 blocks, so the
// whole round is applied at once as B <- J^T B J, one 2x2 block per task. The
// rotation formulae, skip threshold (0.1 tol), stopping rule
// (max |off-diagonal| <= 1e-14 ||A||_F) and sweep cap (50) are the reference's.
// B (and V when it fits) live in shared memory; otherwise in the L2-resident
// `work` buffer.
__global__ void __launch_bounds__(kJacobiThreads) jacobi_kernel(double* a, index_t l, double* evals,
                                                                double* evecs, double* work,
                                                                int b_in_smem, int v_in_smem,
                                                                int* status, double* gap) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  const index_t npairs = (l + 1) / 2;
  // per-round pair table
  __shared__ int pp[512], qq[512];
  __shared__ double cs[512], sn[512], tt[512];
  __shared__ int act[512];
  double* B = b_in_smem ? smem : work;
  double* V = v_in_smem ? (b_in_smem ? smem + l * l : smem) : work + l * l;
  const int tid = threadIdx.x;
  const index_t ll = l * l;

  // Copy in with exact symmetry (upper triangle mirrored, jacobi.cpp:54-56),
  // checking the input symmetry like the reference (1e-10 ||A||_F).
  double fro = 0.0, asym = 0.0;
  for (index_t e = tid; e < ll; e += kJacobiThreads) {
    const index_t j = e / l, i = e % l;
    const double v = a[e];
    fro += v * v;
    asym = fmax(asym, fabs(v - a[i * l + j]));
    B[e] = i <= j ? v : a[i * l + j];
    V[e] = i == j ? 1.0 : 0.0;
  }
  block_sum_reduce(fro, red);
  block_max_reduce(asym, red);
  const double fnorm = sqrt(fro);
  if (asym > 1e-10 * fnorm) {
    if (tid == 0) {
      status[0] = 2;
      gap[0] = asym;
    }
    return;
  }
  const double tol = 1e-14 * fnorm;
  const double skip_tol = 0.1 * tol;
  const index_t players = l % 2 == 0 ? l : l + 1;

  auto max_off = [&]() {
    double w = 0.0;
    for (index_t e = tid; e < ll; e += kJacobiThreads) {
      const index_t j = e / l, i = e % l;
      if (i < j) w = fmax(w, fabs(B[e]));
    }
    block_max_reduce(w, red);
    return w;
  };

  double off = max_off();
  int sweep = 0;
  while (off > tol) {
    if (sweep++ >= kMaxSweeps) {
      if (tid == 0) {
        status[0] = 1;
        gap[0] = off;
      }
      return;
    }
    for (index_t round = 0; round < players - 1; ++round) {
      // 1. rotation for each pair of this round
      for (index_t k = tid; k < players / 2; k += kJacobiThreads) {
        index_t x = k == 0 ? players - 1 : (round + k) % (players - 1);
        index_t y = (round + players - 1 - k) % (players - 1);
        if (x >= l || y >= l) {  // bye: a single index with identity rotation
          pp[k] = static_cast<int>(x < l ? x : y);
          qq[k] = -1;
          act[k] = 0;
          continue;
        }
        if (x > y) {
          const index_t t = x;
          x = y;
          y = t;
        }
        pp[k] = static_cast<int>(x);
        qq[k] = static_cast<int>(y);
        const double apq = B[y * l + x];
        if (fabs(apq) <= skip_tol) {
          act[k] = 0;
          continue;
        }
        const double app = B[x * l + x], aqq = B[y * l + y];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = theta >= 0.0 ? 1.0 / (theta + sqrt(theta * theta + 1.0))
                                      : -1.0 / (-theta + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        act[k] = 1;
        cs[k] = c;
        sn[k] = t * c;
        tt[k] = t;
      }
      __syncthreads();
      // 2. B <- J^T B J over 2x2 blocks (P <= Q; the (Q, P) block is its transpose)
      const index_t nblocks = npairs * (npairs + 1) / 2;
      for (index_t e = tid; e < nblocks; e += kJacobiThreads) {
        // unrank e -> (P, Q), P <= Q, row-major over the upper triangle
        index_t P = static_cast<index_t>((2.0 * npairs + 1.0 -
                                          sqrt((2.0 * npairs + 1.0) * (2.0 * npairs + 1.0) - 8.0 * e)) /
                                         2.0);
        if (P < 0) P = 0;
        while (P > 0 && P * npairs - P * (P - 1) / 2 > e) --P;
        while ((P + 1) * npairs - (P + 1) * P / 2 <= e) ++P;
        const index_t Q = P + (e - (P * npairs - P * (P - 1) / 2));
        const bool aP = act[P], aQ = act[Q];
        if (!aP && !aQ) continue;
        const int p1 = pp[P], q1 = qq[P], p2 = pp[Q], q2 = qq[Q];
        if (P == Q) {  // diagonal block: the reference's closed form
          const double apq = B[q1 * l + p1];
          const double t = tt[P];
          B[p1 * l + p1] = B[p1 * l + p1] - t * apq;
          B[q1 * l + q1] = B[q1 * l + q1] + t * apq;
          B[q1 * l + p1] = 0.0;
          B[p1 * l + q1] = 0.0;
          continue;
        }
        const double c1 = aP ? cs[P] : 1.0, s1 = aP ? sn[P] : 0.0;
        const double c2 = aQ ? cs[Q] : 1.0, s2 = aQ ? sn[Q] : 0.0;
        // rows {p1, q1} x cols {p2, q2}; q = -1 marks a bye (single index)
        double b00 = B[p2 * l + p1];
        double b01 = q2 >= 0 ? B[q2 * l + p1] : 0.0;
        double b10 = q1 >= 0 ? B[p2 * l + q1] : 0.0;
        double b11 = (q1 >= 0 && q2 >= 0) ? B[q2 * l + q1] : 0.0;
        // columns (B J)
        double n00 = c2 * b00 - s2 * b01, n01 = s2 * b00 + c2 * b01;
        double n10 = c2 * b10 - s2 * b11, n11 = s2 * b10 + c2 * b11;
        // rows (J^T B J)
        b00 = c1 * n00 - s1 * n10;
        b10 = s1 * n00 + c1 * n10;
        b01 = c1 * n01 - s1 * n11;
        b11 = s1 * n01 + c1 * n11;
        B[p2 * l + p1] = b00;
        B[p1 * l + p2] = b00;
        if (q2 >= 0) {
          B[q2 * l + p1] = b01;
          B[p1 * l + q2] = b01;
        }
        if (q1 >= 0) {
          B[p2 * l + q1] = b10;
          B[q1 * l + p2] = b10;
        }
        if (q1 >= 0 && q2 >= 0) {
          B[q2 * l + q1] = b11;
          B[q1 * l + q2] = b11;
        }
      }
      // 3. V <- V J (jacobi.cpp:107-114)
      for (index_t e = tid; e < npairs * l; e += kJacobiThreads) {
        const index_t P = e / l, i = e % l;
        if (!act[P]) continue;
        const int p = pp[P], q = qq[P];
        const double c = cs[P], s = sn[P];
        const double x = V[p * l + i], y = V[q * l + i];
        V[p * l + i] = c * x - s * y;
        V[q * l + i] = s * x + c * y;
      }
      __syncthreads();
    }
    off = max_off();
  }
  // Stable descending order of the diagonal (jacobi.cpp:119-133).
  for (index_t i = tid; i < l; i += kJacobiThreads) {
    const double di = B[i * l + i];
    index_t rank = 0;
    for (index_t j = 0; j < l; ++j) {
      const double dj = B[j * l + j];
      rank += (dj > di) || (dj == di && j < i);
    }
    evals[rank] = di;
    for (index_t r = 0; r < l; ++r) evecs[rank * l + r] = V[i * l + r];
  }
  if (tid == 0) {
    status[0] = 0;
    status[1] = sweep;
    gap[0] = off;
  }
}


// V(j, r) = (sum_i F(i, j) U~(i, r)) / sigma_r, i ascending, separate mul/add
// (truncated_svd.cpp:52-62); sigma_r = sqrt(lambda_r).
// V = F^T U~ diag(sigma)^{-1} (truncated_svd.cpp:51-62): each dot product runs
// over i in ascending order with separate multiply and add (the reference's
// rounding), tiled 32 (j) x 32 (r) per CTA through shared memory so F and U~
// are read once per tile instead of once per output.
__global__ void __launch_bounds__(256) vform_kernel(const double* __restrict__ f, index_t l, index_t n,
                                                    const double* __restrict__ ut,
                                                    const double* __restrict__ evals, index_t k,
                                                    double* __restrict__ sigma, double* __restrict__ v) {
  __shared__ double fs[32][33];
  __shared__ double us[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const index_t j0 = static_cast<index_t>(blockIdx.x) * 32, r0 = static_cast<index_t>(blockIdx.y) * 32;
  if (sigma && blockIdx.x == 0) {
    const index_t e = r0 + ty * 32 + tx;
    if (e < k && ty < 1) sigma[e] = sqrt(evals[e]);
  }
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (index_t i0 = 0; i0 < l; i0 += 32) {
    for (int t = ty; t < 32; t += 8) {
      const index_t j = j0 + t, i = i0 + tx, r = r0 + t;
      fs[tx][t] = (j < n && i < l) ? f[j * l + i] : 0.0;   // fs[i][j]
      us[tx][t] = (r < k && i < l) ? ut[r * l + i] : 0.0;  // us[i][r]
    }
    __syncthreads();
    const int iend = static_cast<int>(l - i0 < 32 ? l - i0 : 32);
    for (int ii = 0; ii < iend; ++ii) {
      const double fv = fs[ii][tx];
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[t] = __dadd_rn(acc[t], __dmul_rn(fv, us[ii][ty + 8 * t]));
    }
    __syncthreads();
  }
  const index_t j = j0 + tx;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const index_t r = r0 + ty + 8 * t;
    if (j < n && r < k) v[r * n + j] = acc[t] / sqrt(evals[r]);
  }
}

// Canonical signs (truncated_svd.cpp:64-80): in each V column the entry of
// largest magnitude (first index on ties) is made non-negative; U~ follows.
__global__ void sign_canon_kernel(double* v, index_t n, double* ut, index_t l) {
  __shared__ double bm[32];
  __shared__ index_t bi[32];
  __shared__ int flip;
  const index_t r = blockIdx.x;
  double* col = v + r * n;
  double best = -1.0;
  index_t arg = 0;
  for (index_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double mag = fabs(col[j]);
    if (mag > best) {
      best = mag;
      arg = j;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const index_t oi = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oi < arg)) {
      best = ob;
      arg = oi;
    }
  }
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    bm[w] = best;
    bi[w] = arg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < static_cast<int>(blockDim.x / 32); ++q)
      if (bm[q] > best || (bm[q] == best && bi[q] < arg)) {
        best = bm[q];
        arg = bi[q];
      }
    flip = col[arg] < 0.0;
  }
  __syncthreads();
  if (!flip) return;
  for (index_t j = threadIdx.x; j < n; j += blockDim.x) col[j] = -col[j];
  if (ut)
    for (index_t i = threadIdx.x; i < l; i += blockDim.x) ut[r * l + i] = -ut[r * l + i];
}

// Cholesky of G (lazy_projector.cpp:12-37: pivot tolerance 1e-14 * max diag,
// RankDeficiencyError at the first failing pivot) and the inverse of L,
// written as w[j * l + c] = L^{-1}(j, c) — i.e. W = R^{-1} = L^{-T} as an
// x-times-W operand of the sketch GEMM. Blocked right-looking: a one-CTA panel
// factorisation of 32 columns in shared memory, then the trailing SYRK update
// over 32 x 32 tiles on many CTAs; the inverse by one warp per column of
// L^{-1} (forward substitution, axpy form). The reference sums left-looking;
// the orders differ by roundoff only.
constexpr int kCholNb = 32;

__global__ void chol_copy_kernel(const double* __restrict__ g, index_t l, double* __restrict__ lm) {
  const index_t e = static_cast<index_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= l * l) return;
  const index_t c = e / l, r = e % l;
  lm[e] = r >= c ? g[e] : 0.0;
}

// Panel [p0, p0 + nb) x rows [p0, l): factor in shared memory (or in place
// when the panel exceeds it, in_smem = 0), write back.
__global__ void __launch_bounds__(256) chol_panel_kernel(const double* __restrict__ g, index_t l, index_t p0,
                                                         double* __restrict__ lm, int* status, int in_smem,
                                                         double tol_rel) {
  extern __shared__ double psh[];  // [nb][rows] column-major panel
  __shared__ double red[32];
  __shared__ int fail;
  if (status[0] != 0) return;  // an earlier panel failed
  const int nb = static_cast<int>(l - p0 < kCholNb ? l - p0 : kCholNb);
  const index_t rows = l - p0;
  double* pan = in_smem ? psh : lm + p0 * l + p0;
  const index_t ldp = in_smem ? rows : l;
  double maxd = 0.0;
  for (index_t j = threadIdx.x; j < l; j += blockDim.x) maxd = fmax(maxd, g[j * l + j]);
  block_max_reduce(maxd, red);
  const double tol = tol_rel * maxd;
  if (threadIdx.x == 0) fail = 0;
  if (in_smem) {
    for (index_t e = threadIdx.x; e < rows * nb; e += blockDim.x) {
      const index_t j = e / rows, r = e % rows;
      pan[e] = lm[(p0 + j) * l + p0 + r];
    }
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    double* cj = pan + static_cast<index_t>(j) * ldp;
    const double d = cj[j];
    if (!(d > tol)) {  // (NaN fails too)
      if (threadIdx.x == 0) fail = static_cast<int>(p0 + j) + 1;
      break;
    }
    const double dj = sqrt(d), inv = 1.0 / dj;
    __syncthreads();  // everyone has read cj[j]
    for (index_t r = j + threadIdx.x; r < rows; r += blockDim.x) cj[r] = r == j ? dj : cj[r] * inv;
    __syncthreads();
    // rank-1 update of the panel's remaining columns (rows >= column)
    for (int k = j + 1; k < nb; ++k) {
      double* ck = pan + static_cast<index_t>(k) * ldp;
      const double lkj = cj[k];
      for (index_t r = k + threadIdx.x; r < rows; r += blockDim.x) ck[r] -= cj[r] * lkj;
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail) {
    if (threadIdx.x == 0) status[0] = fail;
    return;
  }
  if (in_smem) {
    for (index_t e = threadIdx.x; e < rows * nb; e += blockDim.x) {
      const index_t j = e / rows, r = e % rows;
      if (r >= j) lm[(p0 + j) * l + p0 + r] = pan[e];
    }
  }
}

// Trailing update A(i, k) -= sum_{j in panel} L(i, j) L(k, j) for i >= k >= p0 + nb.
__global__ void __launch_bounds__(256) chol_syrk_kernel(index_t l, index_t p0, double* __restrict__ lm,
                                                        const int* status) {
  if (status[0] != 0) return;
  const index_t t0 = p0 + kCholNb;
  const index_t i0 = t0 + static_cast<index_t>(blockIdx.x) * 32, k0 = t0 + static_cast<index_t>(blockIdx.y) * 32;
  if (blockIdx.x < blockIdx.y) return;  // upper tiles
  __shared__ double li[kCholNb][33];
  __shared__ double lk[kCholNb][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  for (int j = ty; j < kCholNb; j += 8) {
    const index_t c = p0 + j;
    li[j][tx] = i0 + tx < l ? lm[c * l + i0 + tx] : 0.0;
    lk[j][tx] = k0 + tx < l ? lm[c * l + k0 + tx] : 0.0;
  }
  __syncthreads();
  for (int q = 0; q < 4; ++q) {
    const index_t i = i0 + tx, k = k0 + ty + 8 * q;
    if (i >= l || k >= l || i < k) continue;
    double acc = 0.0;
#pragma unroll 8
    for (int j = 0; j < kCholNb; ++j) acc = fma(li[j][tx], lk[j][ty + 8 * q], acc);
    lm[k * l + i] -= acc;
  }
}

// W = L^{-T}: warp per column c of L^{-1}; the right-hand side (e_c) in shared
// memory, reciprocal diagonal precomputed.
__global__ void __launch_bounds__(256) chol_inv_kernel(const double* __restrict__ lm, index_t l, double* __restrict__ w,
                                                       int* status) {
  extern __shared__ double sh[];
  if (status[0] != 0) return;
  double* dinv = sh;                                            // [l]
  double* b = sh + l + static_cast<index_t>(threadIdx.x / 32) * l;  // this warp's [l]
  for (index_t j = threadIdx.x; j < l; j += blockDim.x) dinv[j] = 1.0 / lm[j * l + j];
  __syncthreads();
  const int lane = threadIdx.x % 32;
  const index_t c = static_cast<index_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  if (c >= l) return;
  for (index_t r = lane; r < l; r += 32) b[r] = r == c ? 1.0 : 0.0;
  __syncwarp();
  for (index_t j = c; j < l; ++j) {
    const double x = b[j] * dinv[j];  // L^{-1}(j, c)
    if (lane == 0) w[j * l + c] = x;
    const double* colj = lm + j * l;
    for (index_t r = j + 1 + lane; r < l; r += 32) b[r] -= colj[r] * x;
    __syncwarp();
  }
  for (index_t j = lane; j < c; j += 32) w[j * l + c] = 0.0;
  if (c == 0 && lane == 0) status[0] = 0;
}

constexpr int kCholRows = 8, kCholMaxL = 256;  // one-CTA kernels: rows per lane, l <= 256

// chol_inv_kernel with L's packed lower triangle staged in shared memory once
// per CTA (l <= ~220 with 8 warps): the column walk reads L(r, j) at shared-memory
// latency instead of L1/L2's (the global variant: 0.11 ms at l = 220). Same
// arithmetic in the same order.
__global__ void __launch_bounds__(256) chol_inv_smem_kernel(const double* __restrict__ lm, index_t l,
                                                            double* __restrict__ w, int* status) {
  extern __shared__ double sh[];
  if (status[0] != 0) return;
  const int L = static_cast<int>(l), lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* dinv = sh;                                 // [l]
  double* b = sh + L + wid * L;                      // this warp's [l]
  double* tri = sh + L + (blockDim.x >> 5) * L;      // packed lower triangle, column j at tri + off(j)
  auto off = [&](int j) { return j * L - j * (j - 1) / 2 - j; };
  for (int j = threadIdx.x; j < L; j += blockDim.x) dinv[j] = 1.0 / lm[static_cast<index_t>(j) * l + j];
  for (int j = wid; j < L; j += blockDim.x >> 5) {  // a lane's rows of a column loaded together
    double v[kCholRows];
#pragma unroll
    for (int t = 0; t < kCholRows; ++t) {
      const int r = j + lane + 32 * t;
      v[t] = r < L ? lm[static_cast<index_t>(j) * l + r] : 0.0;
    }
    double* cj = tri + off(j);
#pragma unroll
    for (int t = 0; t < kCholRows; ++t)
      if (j + lane + 32 * t < L) cj[j + lane + 32 * t] = v[t];
  }
  __syncthreads();
  const int c = static_cast<int>(blockIdx.x) * (blockDim.x >> 5) + wid;
  if (c >= L) return;
  for (int r = lane; r < L; r += 32) b[r] = r == c ? 1.0 : 0.0;
  __syncwarp();
  for (int j = c; j < L; ++j) {
    const double x = b[j] * dinv[j];  // L^{-1}(j, c)
    if (lane == 0) w[static_cast<index_t>(j) * l + c] = x;
    const double* colj = tri + off(j);
    for (int r = j + 1 + lane; r < L; r += 32) b[r] -= colj[r] * x;
    __syncwarp();
  }
  for (int j = lane; j < c; j += 32) w[static_cast<index_t>(j) * l + c] = 0.0;
  if (c == 0 && lane == 0) status[0] = 0;
}

// tmp(r, j) = sum_{s <= r} L^{-1}(r, s) F(s, j), tiled: a CTA computes 64 r x
// 64 j outputs from 16-wide slabs of L^{-1} rows and F columns in shared memory,
// 4 x 4 per thread; each output still sums s = 0, 1, ... in order with FMAs
// (the zero entries above the diagonal add nothing), as the untiled kernel did.
__global__ void __launch_bounds__(256) apply_linv_tiled_kernel(const double* __restrict__ w, index_t l,
                                                                const double* __restrict__ f, index_t n,
                                                                double* __restrict__ out) {
  __shared__ double ws[16][65];  // [s][r]
  __shared__ double fs[16][65];  // [s][j]
  const index_t r0 = static_cast<index_t>(blockIdx.x) * 64, j0 = static_cast<index_t>(blockIdx.y) * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // r = r0 + ty + 16 a, j = j0 + tx + 16 b
  double acc[4][4] = {};
  const index_t s_end = r0 + 64 < l ? r0 + 64 : l;
  for (index_t s0 = 0; s0 < s_end; s0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int k = e % 16, i = e / 16;
      const index_t r = r0 + i, sv = s0 + k;
      ws[k][i] = (r < l && sv <= r) ? w[r * l + sv] : 0.0;
      const index_t j = j0 + i;
      fs[k][i] = (j < n && sv < l) ? f[j * l + sv] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = ws[k][ty + 16 * q];
        b[q] = fs[k][tx + 16 * q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[q][p] = fma(a[q], b[p], acc[q][p]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const index_t r = r0 + ty + 16 * q, j = j0 + tx + 16 * p;
      if (r < l && j < n) out[j * l + r] = acc[q][p];
    }
}


}  // namespace

void launch_gram(cudaStream_t s, const double* f, index_t l, index_t n, double* g) {
  const index_t total = l * l;
  gram_kernel<<<static_cast<unsigned>(ceil_div(total, 128)), 128, 0, s>>>(f, l, n, g);
}

namespace {
// G partial for one n-chunk: 64 x 64 output tile, DFMA, 4 x 4 per thread.
__global__ void __launch_bounds__(256) gram_split_kernel(const double* __restrict__ f, int l, int n, int chunk,
                                                         double* __restrict__ part) {
  constexpr int T = 64, BK = 16;
  __shared__ double As[BK][T + 1];
  __shared__ double Bs[BK][T + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int i0 = blockIdx.x * T, j0 = blockIdx.y * T;
  const int c = blockIdx.z;
  const int k_begin = c * chunk, k_end = min(n, k_begin + chunk);
  double acc[4][4] = {};
  for (int k0 = k_begin; k0 < k_end; k0 += BK) {
    for (int idx = threadIdx.x; idx < T * BK; idx += 256) {
      const int ii = idx % T, kk = idx / T;  // consecutive threads -> consecutive rows of F
      const int gk = k0 + kk;
      As[kk][ii] = (i0 + ii < l && gk < k_end) ? f[static_cast<size_t>(gk) * l + i0 + ii] : 0.0;
      Bs[kk][ii] = (j0 + ii < l && gk < k_end) ? f[static_cast<size_t>(gk) * l + j0 + ii] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = As[kk][ty + 16 * q];
        bv[q] = Bs[kk][tx + 16 * q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(av[p], bv[q], acc[p][q]);
    }
    __syncthreads();
  }
  double* dst = part + static_cast<size_t>(c) * l * l;
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gi = i0 + ty + 16 * p, gj = j0 + tx + 16 * q;
      if (gi < l && gj < l) dst[static_cast<size_t>(gj) * l + gi] = acc[p][q];
    }
}
}  // namespace

index_t gram_fast_chunks(index_t l, index_t n) {
  const index_t tiles = ceil_div(l, 64) * ceil_div(l, 64);
  index_t chunks = ceil_div(2 * 148, tiles);
  const index_t max_chunks = ceil_div(n, 64);
  return chunks < max_chunks ? (chunks < 1 ? 1 : chunks) : max_chunks;
}

void launch_gram_fast(cudaStream_t s, const double* f, index_t l, index_t n, double* g, double* part) {
  const index_t chunks = gram_fast_chunks(l, n);
  const index_t chunk = round_up(ceil_div(n, chunks), 16);
  const index_t nch = ceil_div(n, chunk);
  dim3 grid(static_cast<unsigned>(ceil_div(l, 64)), static_cast<unsigned>(ceil_div(l, 64)),
            static_cast<unsigned>(nch));
  gram_split_kernel<<<grid, 256, 0, s>>>(f, static_cast<int>(l), static_cast<int>(n), static_cast<int>(chunk),
                                         nch == 1 ? g : part);
  if (nch > 1) launch_reduce_partials(s, part, nch, l * l, g);
}

void launch_jacobi_eigh(cudaStream_t s, double* a, index_t l, double* evals, double* evecs,
                        double* work, int* status, double* gap) {
  if (l > 1024) throw Error(kInvalidArgument, "eigh: l > 1024 is not supported on the device");
  const std::size_t mat = static_cast<std::size_t>(l * l) * sizeof(double);
  const std::size_t cap = 200 * 1024;
  int b_smem = mat <= cap ? 1 : 0;
  int v_smem = (b_smem && 2 * mat <= cap) ? 1 : 0;
  const std::size_t smem = static_cast<std::size_t>(b_smem + v_smem) * mat;
  LPCA_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem > 0 ? smem : 16)));
  jacobi_kernel<<<1, kJacobiThreads, smem, s>>>(a, l, evals, evecs, work, b_smem, v_smem, status, gap);
}

void launch_vform(cudaStream_t s, const double* f, index_t l, index_t n, const double* ut,
                  const double* evals, index_t k, double* sigma, double* v) {
  const index_t total = n * k > k ? n * k : k;
  (void)total;
  const dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(k, 32)));
  vform_kernel<<<grid, dim3(32, 8), 0, s>>>(f, l, n, ut, evals, k, sigma, v);
}

void launch_sign_canon(cudaStream_t s, double* v, index_t n, index_t k, double* ut, index_t l) {
  sign_canon_kernel<<<static_cast<unsigned>(k), 256, 0, s>>>(v, n, ut, l);
}

namespace {
// The whole Cholesky factorisation in one CTA when the lower triangle fits
// shared memory (l <= ~236): packed columns, right-looking, blocked by panels
// of kCholPanel columns. Within a panel one barrier per column (the update runs
// on the unscaled column j: A(r, c) -= A(r, j) (A(c, j) / d), d = A(j, j), for
// the panel's later columns only); the panel is then scaled to L and the
// trailing matrix takes one rank-kCholPanel update, a warp per kCholGroup
// columns with lanes down the rows and the panel's rows L(r, :) in registers,
// so each trailing element is read and written once per panel instead of once
// per column (the column-at-a-time kernel was bound by shared-memory traffic:
// 0.37 ms at l = 220). Same pivot rule and status as the panel path (the first
// column whose pivot fails, 1-based); L goes to lm (column-major, zeros above)
// for chol_inv_kernel.
constexpr int kCholPanel = 8, kCholGroup = 2;

__global__ void __launch_bounds__(512) chol_small_kernel(const double* __restrict__ g, index_t l, double tol_rel,
                                                          double* __restrict__ lm, int* status) {
  extern __shared__ double tri[];  // packed lower triangle, column-major: column c at coff(c)
  __shared__ double red[32];
  __shared__ int coff[kCholMaxL];    // col(c)[r] = A(r, c), r >= c
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int L = static_cast<int>(l);
  for (int c = tid; c < L; c += blockDim.x) coff[c] = c * L - c * (c - 1) / 2 - c;
  __syncthreads();
  auto col = [&](int c) { return tri + coff[c]; };
  double maxd = 0.0;
  for (index_t j = tid; j < l; j += blockDim.x) maxd = fmax(maxd, g[j * l + j]);
  block_max_reduce(maxd, red);
  const double tol = tol_rel * maxd;
  // a lane's rows of a column loaded together (one L2 latency per column, not per row)
  for (int c = warp; c < L; c += nw) {
    double v[kCholRows];
#pragma unroll
    for (int t = 0; t < kCholRows; ++t) {
      const int r = c + lane + 32 * t;
      v[t] = r < L ? g[static_cast<index_t>(c) * l + r] : 0.0;
    }
    double* cc = col(c);
#pragma unroll
    for (int t = 0; t < kCholRows; ++t)
      if (c + lane + 32 * t < L) cc[c + lane + 32 * t] = v[t];
  }
  __syncthreads();
  int fail_at = 0;
  for (int p0 = 0; p0 < L && !fail_at; p0 += kCholPanel) {
    const int pe = p0 + kCholPanel < L ? p0 + kCholPanel : L;
    for (int j = p0; j < pe; ++j) {
      const double* cj = col(j);
      const double d = cj[j];
      if (!(d > tol)) {  // (NaN fails too); every thread tests: a uniform break
        fail_at = j + 1;
        break;
      }
      const double inv_d = 1.0 / d;
      for (int c = j + 1 + warp; c < pe; c += nw) {
        double* cc = col(c);
        const double ljc = cj[c] * inv_d;
        // all of the lane's loads before its stores (at most kCholRows rows per
        // lane): one shared-memory latency per column instead of one per row
        double a[kCholRows], b[kCholRows];
#pragma unroll
        for (int t = 0; t < kCholRows; ++t) {
          const int r = c + lane + 32 * t;
          a[t] = r < L ? cj[r] : 0.0;
          b[t] = r < L ? cc[r] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < kCholRows; ++t) {
          const int r = c + lane + 32 * t;
          if (r < L) cc[r] = fma(-a[t], ljc, b[t]);
        }
      }
      __syncthreads();
    }
    if (fail_at) break;
    for (int j = p0 + warp; j < pe; j += nw) {  // the panel becomes L
      double* cj = col(j);
      const double sq = sqrt(cj[j]), isq = 1.0 / sq;
      for (int r = j + 1 + lane; r < L; r += 32) cj[r] *= isq;
      if (lane == 0) cj[j] = sq;
    }
    __syncthreads();
    const int np = pe - p0, ngroups = (L - pe + kCholGroup - 1) / kCholGroup;
    const double* pk[kCholPanel];  // the panel's columns
#pragma unroll
    for (int k = 0; k < kCholPanel; ++k) pk[k] = col(k < np ? p0 + k : p0);
    for (int grp = warp; grp < ngroups; grp += nw) {
      const int c0 = pe + grp * kCholGroup;
      double* cq[kCholGroup];
#pragma unroll
      for (int q = 0; q < kCholGroup; ++q) cq[q] = col(c0 + q < L ? c0 + q : c0);
      double lc[kCholGroup][kCholPanel];
#pragma unroll
      for (int q = 0; q < kCholGroup; ++q)
#pragma unroll
        for (int k = 0; k < kCholPanel; ++k) lc[q][k] = (c0 + q < L && k < np) ? pk[k][c0 + q] : 0.0;
      // two rows per lane at a time, every load before the stores
      for (int r0 = c0 + lane; r0 < L; r0 += 64) {
        double lr[2][kCholPanel], v[2][kCholGroup];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + 32 * h;
#pragma unroll
          for (int k = 0; k < kCholPanel; ++k) lr[h][k] = (k < np && r < L) ? pk[k][r] : 0.0;
#pragma unroll
          for (int q = 0; q < kCholGroup; ++q) v[h][q] = (r < L && r >= c0 + q) ? cq[q][r] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + 32 * h;
#pragma unroll
          for (int q = 0; q < kCholGroup; ++q) {
            if (r >= L || r < c0 + q) continue;  // (also covers c0 + q >= L)
            double t = v[h][q];
#pragma unroll
            for (int k = 0; k < kCholPanel; ++k) t = fma(-lr[h][k], lc[q][k], t);
            cq[q][r] = t;
          }
        }
      }
    }
    __syncthreads();
  }
  if (fail_at) {
    if (tid == 0) status[0] = fail_at;
    return;
  }
  for (int c = warp; c < L; c += nw) {
    const double* cc = col(c);
    for (int r = lane; r < L; r += 32) lm[static_cast<index_t>(c) * l + r] = r >= c ? cc[r] : 0.0;
  }
}
}  // namespace

namespace {
// W = L^{-T} of lm (launch_chol_inverse's layout): the shared-memory variant when
// L's packed triangle, dinv and the warps' right-hand sides fit one CTA.
void launch_chol_inv(cudaStream_t s, const double* lm, index_t l, double* w, int* status) {
  const std::size_t packed = static_cast<std::size_t>(l) * (l + 1) / 2;
  const std::size_t sm8 = (static_cast<std::size_t>(l) * 9 + packed) * sizeof(double);
  if (sm8 <= 227 * 1024) {
    LPCA_CUDA(cudaFuncSetAttribute(chol_inv_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm8 > 48 * 1024 ? sm8 : 48 * 1024)));
    chol_inv_smem_kernel<<<static_cast<unsigned>(ceil_div(l, 8)), 256, sm8, s>>>(lm, l, w, status);
    return;
  }
  int wpb = 8;  // warps per block: dinv + one right-hand side per warp in shared memory
  while (wpb > 1 && static_cast<std::size_t>(l) * (wpb + 1) * sizeof(double) > 200 * 1024) wpb >>= 1;
  const std::size_t ism = static_cast<std::size_t>(l) * (wpb + 1) * sizeof(double);
  if (ism > 227 * 1024) throw Error(kInternal, "chol_inverse: l too large for the shared-memory solve");
  LPCA_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(ism > 48 * 1024 ? ism : 48 * 1024)));
  chol_inv_kernel<<<static_cast<unsigned>(ceil_div(l, wpb)), 32 * wpb, ism, s>>>(lm, l, w, status);
}
}  // namespace

void launch_chol_inverse(cudaStream_t s, const double* g, index_t l, double* rinv, double* work,
                         int* status, double tol_rel) {
  if (l <= 0) return;
  LPCA_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
  const std::size_t tri_bytes = static_cast<std::size_t>(l) * (l + 1) / 2 * sizeof(double);
  if (tri_bytes <= 220 * 1024) {
    LPCA_CUDA(cudaFuncSetAttribute(chol_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(tri_bytes < 48 * 1024 ? 48 * 1024 : tri_bytes)));
    chol_small_kernel<<<1, 512, tri_bytes, s>>>(g, l, tol_rel, work, status);
  } else {
    chol_copy_kernel<<<static_cast<unsigned>(ceil_div(l * l, 256)), 256, 0, s>>>(g, l, work);
    std::size_t psm = static_cast<std::size_t>(l) * kCholNb * sizeof(double);
    const int in_smem = psm <= 200 * 1024 ? 1 : 0;
    if (!in_smem) psm = 0;
    LPCA_CUDA(cudaFuncSetAttribute(chol_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(psm > 48 * 1024 ? psm : 48 * 1024)));
    for (index_t p0 = 0; p0 < l; p0 += kCholNb) {
      chol_panel_kernel<<<1, 256, psm, s>>>(g, l, p0, work, status, in_smem, tol_rel);
      const index_t t = l - p0 - kCholNb;
      if (t > 0) {
        const unsigned tiles = static_cast<unsigned>(ceil_div(t, 32));
        chol_syrk_kernel<<<dim3(tiles, tiles), 256, 0, s>>>(l, p0, work, status);
      }
    }
  }
  launch_chol_inv(s, work, l, rinv, status);
}

namespace {
// g_ii += c * trace(g): the shift of shifted CholeskyQR (one CTA, fixed-order sum).
__global__ void add_trace_shift_kernel(double* g, index_t l, double c) {
  __shared__ double red[32];
  double t = 0.0;
  for (index_t j = threadIdx.x; j < l; j += blockDim.x) t += g[j * l + j];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const double shift = c * red[0];
  for (index_t j = threadIdx.x; j < l; j += blockDim.x) g[j * l + j] += shift;
}
}  // namespace

namespace {
__global__ void flag_to_f64_kernel(const int* flag, double* out) { out[0] = flag[0] != 0 ? 1.0 : 0.0; }
}  // namespace

void launch_flag_to_f64(cudaStream_t s, const int* flag, double* out) { flag_to_f64_kernel<<<1, 1, 0, s>>>(flag, out); }

void launch_add_trace_shift(cudaStream_t s, double* g, index_t l, double c) {
  add_trace_shift_kernel<<<1, 1024, 0, s>>>(g, l, c);
}

void launch_apply_rinv_t(cudaStream_t s, const double* rinv, index_t l, double* f, index_t n,
                         double* tmp) {
  const index_t total = l * n;
  const dim3 grid(static_cast<unsigned>(ceil_div(l, 64)), static_cast<unsigned>(ceil_div(n, 64)));
  apply_linv_tiled_kernel<<<grid, 256, 0, s>>>(rinv, l, f, n, tmp);
  LPCA_CUDA(cudaMemcpyAsync(f, tmp, static_cast<std::size_t>(total) * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
}

// ---- pieces of shifted CholeskyQR3 (lpca.cu cholqr3) ---------------------------
namespace {
// C = op(A) op(B) + beta C for l x l column-major matrices (op = transpose when
// the flag is set); one thread per output, fixed k order.
__global__ void small_gemm_kernel(int ta, int tb, index_t l, const double* __restrict__ a,
                                  const double* __restrict__ b, double* __restrict__ c, double beta) {
  const index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x;
  if (e >= l * l) return;
  const index_t j = e / l, i = e % l;
  double acc = 0.0;
  for (index_t k = 0; k < l; ++k) {
    const double av = ta ? a[i * l + k] : a[k * l + i];
    const double bv = !b ? (k == j ? 1.0 : 0.0) : tb ? b[k * l + j] : b[j * l + k];  // null B = identity
    acc = fma(av, bv, acc);
  }
  c[e] = beta != 0.0 ? fma(beta, c[e], acc) : acc;
}

// rdiag = diag(R_p) (first pass) or rdiag *= diag(R_p), with diag(R_p) = 1 / W_jj
// for W = R_p^{-1} as launch_chol_inverse writes it.
__global__ void rdiag_update_kernel(const double* __restrict__ w, index_t l, double* __restrict__ rdiag, int first) {
  const index_t j = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x;
  if (j >= l) return;
  const double d = 1.0 / w[j * l + j];
  rdiag[j] = first ? d : rdiag[j] * d;
}

__global__ void trace_kernel(const double* __restrict__ g, index_t l, double* out) {
  __shared__ double red[32];
  double t = 0.0;
  for (index_t j = threadIdx.x; j < l; j += blockDim.x) t += g[j * l + j];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) out[0] = t;
  }
}

// lm (lower, column-major) = R^T for an upper-triangular R; zeros above.
__global__ void upper_to_lower_kernel(const double* __restrict__ r, index_t l, double* __restrict__ lm) {
  const index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x;
  if (e >= l * l) return;
  const index_t c = e / l, i = e % l;
  lm[e] = i >= c ? r[i * l + c] : 0.0;
}
}  // namespace

void launch_small_gemm(cudaStream_t s, int ta, int tb, index_t l, const double* a, const double* b, double* c,
                       double beta) {
  if (l <= 0) return;
  small_gemm_kernel<<<static_cast<unsigned>(ceil_div(l * l, 128)), 128, 0, s>>>(ta, tb, l, a, b, c, beta);
}

void launch_rdiag_update(cudaStream_t s, const double* w, index_t l, double* rdiag, int first) {
  if (l <= 0) return;
  rdiag_update_kernel<<<static_cast<unsigned>(ceil_div(l, 128)), 128, 0, s>>>(w, l, rdiag, first);
}

void launch_trace(cudaStream_t s, const double* g, index_t l, double* out) { trace_kernel<<<1, 1024, 0, s>>>(g, l, out); }

// W = R^{-1} (launch_chol_inverse's layout) of an upper-triangular R.
void launch_upper_inverse(cudaStream_t s, const double* r, index_t l, double* w, double* work, int* status) {
  if (l <= 0) return;
  LPCA_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
  upper_to_lower_kernel<<<static_cast<unsigned>(ceil_div(l * l, 256)), 256, 0, s>>>(r, l, work);
  launch_chol_inv(s, work, l, w, status);
}

}  // namespace lpca
