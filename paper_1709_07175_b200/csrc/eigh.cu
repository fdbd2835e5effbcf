// Symmetric eigendecomposition on the device, the reference's route
// (proj/core/src/tridiag_eigh.cpp:24-217: Householder tridiagonalisation, then
// the tridiagonal eigenproblem, then back-transformation) re-planned for a GPU:
//
//  1. tridiag_kernel    one CTA; the reference's right-to-left Householder
//                       reduction (tridiag_eigh.cpp:24-81) with the matvec and the
//                       rank-2 update spread over 1024 threads; A in shared
//                       memory when it fits. Exact symmetry is kept by separate
//                       multiply/add in the update (the reference relies on it).
//  2. bisect_kernel     eigenvalues of T by Sturm-count multisection: one warp per
//                       eigenvalue, 32 lanes probe 32 points per round (~5 bits per
//                       round instead of bisection's 1), to ulp(||T||).
//  3. invit_kernel      eigenvectors of T by inverse iteration (pivoted tridiagonal
//                       LU), one thread per eigenvalue; eigenvalues closer than a
//                       relative gap of 1e-3 (or both below 1e-10 ||T||) form a
//                       cluster handled by one thread with modified Gram-Schmidt,
//                       so vectors of close eigenvalues stay orthogonal.
//  4. backxform_kernel  Z = P_{l-1} ... P_1 Y, one warp per eigenvector, reflectors
//                       read from where step 1 left them.
// The reference's QL sweep (tridiag_eigh.cpp:108-170) is a sequential
// bulge chase; steps 2-3 replace it with work that is parallel over eigenvalues.
#include <cuda_runtime.h>

#include <cfloat>

#include "kernels.cuh"

namespace lpca {

namespace {

constexpr int kTriThreads = 1024;
constexpr int kRowLanes = 8;  // threads cooperating on one row of the matvec

__device__ __forceinline__ double warp_sum(double v, unsigned mask = 0xffffffffu) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = lane < static_cast<int>(blockDim.x / 32) ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// Two sums in one pass of barriers (red needs 66 doubles).
__device__ void block_sum2(double& a, double& b, double* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  __syncthreads();
  if (lane == 0) {
    red[w] = a;
    red[33 + w] = b;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double sa = lane < static_cast<int>(blockDim.x / 32) ? red[lane] : 0.0;
    double sb = lane < static_cast<int>(blockDim.x / 32) ? red[33 + lane] : 0.0;
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) {
      red[32] = sa;
      red[65] = sb;
    }
  }
  __syncthreads();
  a = red[32];
  b = red[65];
}

__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = lane < static_cast<int>(blockDim.x / 32) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// ---- 1. Householder tridiagonalisation ------------------------------------------------
// On exit: d (diagonal), e (e[i] couples i-1 and i, e[0] = 0), h (Gram factor of
// reflector i, 0 when no reflector was needed) and, in column i of `refl`
// (rows 0..i-1), the scaled Householder vector u_i.
__global__ void __launch_bounds__(kTriThreads) tridiag_kernel(const double* __restrict__ a, int l,
                                                              double* refl, int a_in_smem, double* d,
                                                              double* e, double* h, double* norm_out,
                                                              int* status, double* gap) {
  extern __shared__ double smem[];
  __shared__ double red[66];
  __shared__ double sh_scal[4];
  double* A = a_in_smem ? smem : refl;
  double* u_s = a_in_smem ? smem + static_cast<size_t>(l) * l : smem;  // u, p, q vectors
  double* p_s = u_s + l;
  double* q_s = p_s + l;
  const int tid = threadIdx.x;
  const int ll = l * l;

  double fro = 0.0, asym = 0.0;
  for (int idx = tid; idx < ll; idx += kTriThreads) {
    const int j = idx / l, i = idx % l;
    const double v = a[idx];
    fro += v * v;
    asym = fmax(asym, fabs(v - a[i * l + j]));
    A[idx] = i <= j ? v : a[i * l + j];  // exact symmetry (tridiag_eigh.cpp:189-191)
  }
  fro = block_sum(fro, red);
  asym = block_max(asym, red);
  const double fnorm = sqrt(fro);
  if (asym > 1e-10 * fnorm) {
    if (tid == 0) {
      status[0] = 2;
      gap[0] = asym;
    }
    return;
  }

  for (int i = l - 1; i >= 1; --i) {
    double* ui = A + static_cast<size_t>(i) * l;
    if (i == 1) {
      if (tid == 0) {
        e[1] = ui[0];
        h[1] = 0.0;
      }
      continue;
    }
    // |x| and x^2 sums in one reduction (the reference sums (x/scale)^2; the
    // two differ by roundoff only)
    double pa = 0.0, ps = 0.0;
    for (int k = tid; k < i; k += kTriThreads) {
      const double x = ui[k];
      pa += fabs(x);
      ps += x * x;
    }
    block_sum2(pa, ps, red);
    const double scale = pa;
    if (scale == 0.0) {
      if (tid == 0) {
        e[i] = 0.0;
        h[i] = 0.0;
      }
      continue;
    }
    const double inv = 1.0 / scale;
    const double sigma = ps * inv * inv;
    for (int k = tid; k < i; k += kTriThreads) u_s[k] = ui[k] * inv;
    if (tid == 0) {
      const double f = ui[i - 1] * inv;
      const double g = f >= 0.0 ? -sqrt(sigma) : sqrt(sigma);
      e[i] = scale * g;
      const double hh = sigma - f * g;
      h[i] = hh;
      sh_scal[0] = hh;
      sh_scal[1] = f - g;
    }
    __syncthreads();
    const double hh = sh_scal[0];
    if (tid == 0) u_s[i - 1] = sh_scal[1];  // the reflector's last entry
    __syncthreads();
    // p = A u / h over the active i x i block (A symmetric: row r is column r,
    // contiguous): kRowLanes threads per row; u^T p accumulates alongside.
    double pu = 0.0;
    for (int base = 0; base < i; base += kTriThreads / kRowLanes) {
      const int r = base + tid / kRowLanes, ln = tid % kRowLanes;
      double acc = 0.0;
      if (r < i) {
        const double* ar = A + static_cast<size_t>(r) * l;
        for (int c = ln; c < i; c += kRowLanes) acc = fma(ar[c], u_s[c], acc);
      }
      for (int o = kRowLanes / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (r < i && ln == 0) {
        const double pr = acc / hh;
        p_s[r] = pr;
        pu += u_s[r] * pr;
      }
    }
    const double kk = block_sum(pu, red) / (2.0 * hh);  // its barriers publish p_s
    for (int k = tid; k < i; k += kTriThreads) q_s[k] = p_s[k] - kk * u_s[k];
    __syncthreads();
    // A <- A - u q^T - q u^T on the active block's lower triangle, mirrored:
    // (r, c) and (c, r) get the same value by construction.
    const int tri = i * (i + 1) / 2;
    for (int t = tid; t < tri; t += kTriThreads) {
      // t -> (r, c), c <= r: row r starts at r (r + 1) / 2
      int r = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      if (r * (r + 1) / 2 > t) --r;
      if ((r + 1) * (r + 2) / 2 <= t) ++r;
      const int c = t - r * (r + 1) / 2;
      const double upd = __dadd_rn(__dmul_rn(u_s[r], q_s[c]), __dmul_rn(q_s[r], u_s[c]));
      const double nv = __dsub_rn(A[static_cast<size_t>(c) * l + r], upd);
      A[static_cast<size_t>(c) * l + r] = nv;
      A[static_cast<size_t>(r) * l + c] = nv;
    }
    for (int k = tid; k < i; k += kTriThreads) ui[k] = u_s[k];  // the reflector, for the back-transformation
    __syncthreads();
  }
  double tn = 0.0;
  for (int k = tid; k < l; k += kTriThreads) {
    d[k] = A[static_cast<size_t>(k) * l + k];
    if (k == 0) e[0] = 0.0;
  }
  __syncthreads();
  for (int k = tid; k < l; k += kTriThreads) {
    const double ek = k > 0 ? fabs(e[k]) : 0.0, ek1 = k + 1 < l ? fabs(e[k + 1]) : 0.0;
    tn = fmax(tn, fabs(d[k]) + ek + ek1);
  }
  tn = block_max(tn, red);
  if (a_in_smem) {  // hand the reflectors to the back-transformation
    for (int idx = tid; idx < ll; idx += kTriThreads) refl[idx] = A[idx];
  }
  if (tid == 0) {
    norm_out[0] = tn;
    status[0] = 0;
    gap[0] = 0.0;
  }
}

// ---- 2. multisection ---------------------------------------------------------------------
// Number of eigenvalues of T strictly below x (Sturm sequence of T - x I).
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e, int l,
                                           double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < l; ++i) {
    q = (d[i] - x) - (e[i] * e[i]) / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// One warp per eigenvalue j (descending): ascending index t = l-1-j.
__global__ void bisect_kernel(const double* __restrict__ d, const double* __restrict__ e, int l,
                              const double* __restrict__ tnorm, double* evals) {
  const int lane = threadIdx.x % 32;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (j >= l) return;
  double lo = DBL_MAX, hi = -DBL_MAX, emax2 = 0.0;
  for (int i = 0; i < l; ++i) {
    const double ei = i > 0 ? fabs(e[i]) : 0.0, ei1 = i + 1 < l ? fabs(e[i + 1]) : 0.0;
    lo = fmin(lo, d[i] - ei - ei1);
    hi = fmax(hi, d[i] + ei + ei1);
    emax2 = fmax(emax2, ei * ei);
  }
  const double tn = tnorm[0];
  const double pivmin = DBL_MIN * fmax(1.0, emax2);
  const double abstol = 2.0 * DBL_EPSILON * fmax(tn, DBL_MIN);
  lo -= abstol;
  hi += abstol;
  const int t = l - 1 - j;
  for (int round = 0; round < 40; ++round) {
    const double w = hi - lo;
    if (w <= abstol + 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) break;
    const double x = lo + w * (static_cast<double>(lane + 1) / 33.0);
    const int c = (x > lo && x < hi) ? sturm_count(d, e, l, x, pivmin) : (x <= lo ? 0 : l);
    // first probe whose count exceeds t bounds the eigenvalue from above
    const unsigned above = __ballot_sync(0xffffffffu, c > t);
    const int k = above ? __ffs(above) - 1 : 32;  // probe index
    const double nhi = k < 32 ? __shfl_sync(0xffffffffu, x, k) : hi;
    const double nlo = k > 0 ? __shfl_sync(0xffffffffu, x, k > 0 ? k - 1 : 0) : lo;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) evals[j] = 0.5 * (lo + hi);
}

// ---- 3. inverse iteration ----------------------------------------------------------------
__device__ __forceinline__ double hash_uniform(unsigned j, unsigned i) {
  unsigned long long z = (static_cast<unsigned long long>(j) << 32) ^ i ^ 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// Scratch layout (per thread j, interleaved so a warp's accesses coalesce):
// field f, row i -> scratch[(f * l + i) * l + j]; fields DL, D, DU, DU2, b.
struct Scr {
  double* base;
  int l, j, stride;  // element (f, i) of thread j at base[(f * l + i) * stride + j]
  __device__ double& at(int f, int i) const { return base[(static_cast<size_t>(f) * l + i) * stride + j]; }
};

// (T - lam I) x = b by pivoted LU (the dgttrf/dgttrs recurrences), b overwritten.
__device__ void tri_solve(const double* __restrict__ d, const double* __restrict__ e, int l, double lam,
                          double tiny, const Scr& s, unsigned char* piv) {
  enum { DL = 0, D = 1, DU = 2, DU2 = 3, B = 4 };
  for (int i = 0; i < l; ++i) {
    s.at(D, i) = d[i] - lam;
    if (i + 1 < l) {
      s.at(DL, i) = e[i + 1];
      s.at(DU, i) = e[i + 1];
    }
  }
  for (int i = 0; i + 1 < l; ++i) {
    const double di = s.at(D, i), dli = s.at(DL, i);
    if (fabs(di) >= fabs(dli)) {
      const double piv_d = fabs(di) < tiny ? (di < 0 ? -tiny : tiny) : di;
      s.at(D, i) = piv_d;
      const double fact = dli / piv_d;
      s.at(DL, i) = fact;
      s.at(D, i + 1) -= fact * s.at(DU, i);
      if (i + 2 < l) s.at(DU2, i) = 0.0;
      piv[i] = 0;
    } else {
      const double fact = di / dli;
      s.at(D, i) = dli;
      s.at(DL, i) = fact;
      const double tmp = s.at(DU, i);
      s.at(DU, i) = s.at(D, i + 1);
      s.at(D, i + 1) = tmp - fact * s.at(D, i + 1);
      if (i + 2 < l) {
        s.at(DU2, i) = s.at(DU, i + 1);
        s.at(DU, i + 1) = -fact * s.at(DU, i + 1);
      }
      piv[i] = 1;
    }
  }
  if (fabs(s.at(D, l - 1)) < tiny) s.at(D, l - 1) = s.at(D, l - 1) < 0 ? -tiny : tiny;
  // L solve
  for (int i = 0; i + 1 < l; ++i) {
    if (!piv[i]) {
      s.at(B, i + 1) -= s.at(DL, i) * s.at(B, i);
    } else {
      const double tmp = s.at(B, i);
      s.at(B, i) = s.at(B, i + 1);
      s.at(B, i + 1) = tmp - s.at(DL, i) * s.at(B, i);
    }
  }
  // U solve
  s.at(B, l - 1) /= s.at(D, l - 1);
  if (l > 1) s.at(B, l - 2) = (s.at(B, l - 2) - s.at(DU, l - 2) * s.at(B, l - 1)) / s.at(D, l - 2);
  for (int i = l - 3; i >= 0; --i)
    s.at(B, i) = (s.at(B, i) - s.at(DU, i) * s.at(B, i + 1) - s.at(DU2, i) * s.at(B, i + 2)) / s.at(D, i);
}

__device__ __forceinline__ bool same_cluster(double a, double b, double tn) {
  const double scale = fmax(fabs(a), fabs(b));
  return fabs(a - b) <= 1e-3 * scale || scale <= 1e-13 * tn;
}

// Y (row-major, Y[i * l + j] = component i of eigenvector j of T).
__global__ void invit_kernel(const double* __restrict__ d, const double* __restrict__ e, int l,
                             const double* __restrict__ evals, const double* __restrict__ tnorm,
                             double* __restrict__ scratch, unsigned char* __restrict__ pivs,
                             double* __restrict__ y, int smem_threads) {
  // LU scratch: in shared memory (5 l doubles + l pivots per thread) when the
  // block fits, else the interleaved global buffer.
  extern __shared__ double sh_scr[];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= l) return;
  const double tn = tnorm[0] > 0.0 ? tnorm[0] : 1.0;  // zero matrix: any orthonormal basis
  // only cluster leaders work; they walk their cluster in order
  if (j > 0 && same_cluster(evals[j - 1], evals[j], tn)) return;
  int end = j + 1;
  while (end < l && same_cluster(evals[end - 1], evals[end], tn)) ++end;
  const Scr s = smem_threads ? Scr{sh_scr, l, static_cast<int>(threadIdx.x), smem_threads} : Scr{scratch, l, j, l};
  unsigned char* piv = smem_threads
                           ? reinterpret_cast<unsigned char*>(sh_scr + static_cast<size_t>(5) * l * smem_threads) +
                                 static_cast<size_t>(threadIdx.x) * l
                           : pivs + static_cast<size_t>(j) * l;
  const double tiny = DBL_EPSILON * tn;
  double prev_shift = 0.0;
  for (int jj = j; jj < end; ++jj) {
    double lam = evals[jj];
    if (jj > j && lam >= prev_shift - 10.0 * DBL_EPSILON * fmax(fabs(lam), tn * 1e-6))
      lam = prev_shift - 10.0 * DBL_EPSILON * fmax(fabs(lam), tn * 1e-6);  // separate equal shifts
    prev_shift = lam;
    for (int i = 0; i < l; ++i) s.at(4, i) = hash_uniform(static_cast<unsigned>(jj), static_cast<unsigned>(i));
    for (int it = 0; it < 3; ++it) {
      tri_solve(d, e, l, lam, tiny, s, piv);
      // modified Gram-Schmidt against the cluster's earlier vectors
      for (int pj = j; pj < jj; ++pj) {
        double dot = 0.0;
        for (int i = 0; i < l; ++i) dot += y[static_cast<size_t>(i) * l + pj] * s.at(4, i);
        for (int i = 0; i < l; ++i) s.at(4, i) -= dot * y[static_cast<size_t>(i) * l + pj];
      }
      double mx = 0.0;
      for (int i = 0; i < l; ++i) mx = fmax(mx, fabs(s.at(4, i)));
      if (mx == 0.0) {
        for (int i = 0; i < l; ++i) s.at(4, i) = hash_uniform(static_cast<unsigned>(jj) + 7919u, static_cast<unsigned>(i));
        continue;
      }
      double nrm = 0.0;
      for (int i = 0; i < l; ++i) {
        const double v = s.at(4, i) / mx;
        s.at(4, i) = v;
        nrm += v * v;
      }
      nrm = 1.0 / sqrt(nrm);
      for (int i = 0; i < l; ++i) s.at(4, i) *= nrm;
    }
    for (int i = 0; i < l; ++i) y[static_cast<size_t>(i) * l + jj] = s.at(4, i);
  }
}

// ---- 4. back-transformation --------------------------------------------------------------
// Z = P_{l-1} ... P_1 Y (reflectors applied in construction order i = 1..l-1,
// as tridiag_eigh.cpp:87-103 builds Q). One warp per eigenvector.
__global__ void backxform_kernel(const double* __restrict__ refl, const double* __restrict__ h, int l,
                                 const double* __restrict__ y, double* __restrict__ z) {
  const int lane = threadIdx.x % 32;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (j >= l) return;
  double* zj = z + static_cast<size_t>(j) * l;  // output column j (column-major)
  for (int k = lane; k < l; k += 32) zj[k] = y[static_cast<size_t>(k) * l + j];
  __syncwarp();
  for (int i = 1; i < l; ++i) {
    const double hi = h[i];
    if (hi == 0.0) continue;
    const double* u = refl + static_cast<size_t>(i) * l;
    double dot = 0.0;
    for (int k = lane; k < i; k += 32) dot = fma(u[k], zj[k], dot);
    dot = warp_sum(dot) / hi;
    for (int k = lane; k < i; k += 32) zj[k] = fma(-dot, u[k], zj[k]);
    __syncwarp();
  }
}

// ---- 5. one refinement step (Ogita & Aishima, "Iterative refinement for
// symmetric eigenvalue decomposition", 2018) ------------------------------------------------
// Inverse iteration gives vectors whose mutual orthogonality is only
// eps ||A|| / gap for eigenvalues that are small next to ||A|| (G's spectrum
// spans ~1e12). With R = I - Z^T Z, S = Z^T A Z and lt_i = S_ii / (1 - R_ii):
//   E_ij = (S_ij + lt_j R_ij) / (lt_j - lt_i)  (i != j, separated),
//   E_ij = R_ij / 2                             (diagonal, or a cluster),
// and Z <- Z + Z E. Since E + E^T = R exactly, the update restores
// orthogonality to second order in the input error whatever the rounding in S.
template <bool kTransA>
__global__ void __launch_bounds__(256) dgemm_small(const double* __restrict__ a, const double* __restrict__ b,
                                                   double* __restrict__ c, int l) {
  // C (l x l) = op(A) B, all column-major l x l; op(A) = A^T when kTransA.
  constexpr int T = 64, BK = 16;
  __shared__ double As[BK][T + 1];
  __shared__ double Bs[BK][T + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int i0 = blockIdx.x * T, j0 = blockIdx.y * T;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < l; k0 += BK) {
    for (int idx = threadIdx.x; idx < T * BK; idx += 256) {
      const int kk = idx % BK, ii = idx / BK;
      const int gi = i0 + ii, gk = k0 + kk;
      // op(A)(gi, gk): A^T -> A(gk, gi) = a[gi * l + gk]; A -> a[gk * l + gi]
      double v = 0.0;
      if (gi < l && gk < l) v = kTransA ? a[static_cast<size_t>(gi) * l + gk] : a[static_cast<size_t>(gk) * l + gi];
      As[kk][ii] = v;
      const int gj = j0 + ii;
      Bs[kk][ii] = (gj < l && gk < l) ? b[static_cast<size_t>(gj) * l + gk] : 0.0;
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
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gi = i0 + ty + 16 * p, gj = j0 + tx + 16 * q;
      if (gi < l && gj < l) c[static_cast<size_t>(gj) * l + gi] = acc[p][q];
    }
}

// In: r = Z^T Z, s = Z^T A Z. Out: e (the correction), column-major.
__global__ void oa_correction_kernel(const double* __restrict__ r, const double* __restrict__ s, int l,
                                     const double* __restrict__ tnorm, double* __restrict__ e) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= l * l) return;
  const int j = idx / l, i = idx % l;
  // S and R are symmetrised: E + E^T = R holds only if the (i,j) and (j,i)
  // corrections see the same numbers (rounding makes computed S asymmetric at
  // eps ||A||, which divided by small gaps would reintroduce non-orthogonality).
  const size_t tidx = static_cast<size_t>(i) * l + j;
  const double rij = (i == j ? 1.0 : 0.0) - 0.5 * (r[idx] + r[tidx]);
  const double sij = 0.5 * (s[idx] + s[tidx]);
  if (i == j) {
    e[idx] = 0.5 * rij;
    return;
  }
  // lt = S_ii / (1 - R_ii) with 1 - R_ii = (Z^T Z)_ii = r_ii
  const double lti = s[static_cast<size_t>(i) * l + i] / r[static_cast<size_t>(i) * l + i];
  const double ltj = s[static_cast<size_t>(j) * l + j] / r[static_cast<size_t>(j) * l + j];
  const double tn = fmax(tnorm[0], DBL_MIN);
  const double scale = fmax(fabs(lti), fabs(ltj));
  const bool cluster = fabs(ltj - lti) <= 1e-3 * scale || scale <= 1e-13 * tn;
  e[idx] = cluster ? 0.5 * rij : (sij + ltj * rij) / (ltj - lti);
}

__global__ void add_kernel(double* __restrict__ z, const double* __restrict__ dz, int count) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < count) z[idx] += dz[idx];
}

}  // namespace

std::size_t eigh_tridiag_workspace(index_t l) {
  // refl (l^2) + y (l^2) + scratch (5 l^2) + d, e, h, norm (3 l + 8) doubles, pivots l^2 bytes
  return static_cast<std::size_t>(7 * l * l + 3 * l + 8) * sizeof(double) + static_cast<std::size_t>(l * l) + 64;
}

void launch_eigh_tridiag(cudaStream_t s, const double* a, index_t l, double* evals, double* evecs, void* work,
                         int* status, double* gap) {
  if (l < 1) return;
  double* w = static_cast<double*>(work);
  double* refl = w;
  double* y = refl + l * l;
  double* scratch = y + l * l;
  double* d = scratch + 5 * l * l;
  double* e = d + l;
  double* h = e + l;
  double* tn = h + l;
  unsigned char* piv = reinterpret_cast<unsigned char*>(tn + 8);
  const std::size_t amat = static_cast<std::size_t>(l * l) * sizeof(double);
  const std::size_t vecs = static_cast<std::size_t>(3 * l) * sizeof(double);
  const int a_smem = amat + vecs <= 200 * 1024 ? 1 : 0;
  const std::size_t smem = (a_smem ? amat : 0) + vecs;
  LPCA_CUDA(cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  tridiag_kernel<<<1, kTriThreads, smem, s>>>(a, static_cast<int>(l), refl, a_smem, d, e, h, tn, status, gap);
  const int warps_per_block = 4;
  const unsigned gblocks = static_cast<unsigned>(ceil_div(l, warps_per_block));
  bisect_kernel<<<gblocks, 32 * warps_per_block, 0, s>>>(d, e, static_cast<int>(l), tn, evals);
  int it = 32;
  while (it > 1 && static_cast<std::size_t>(it) * (40 * l + l) > 200 * 1024) it >>= 1;
  const bool smem_ok = static_cast<std::size_t>(it) * (40 * l + l) <= 200 * 1024;
  const int ithreads = smem_ok ? it : 64;
  const std::size_t ismem = smem_ok ? static_cast<std::size_t>(it) * (40 * l + l) + 16 : 0;
  LPCA_CUDA(cudaFuncSetAttribute(invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ismem)));
  invit_kernel<<<static_cast<unsigned>(ceil_div(l, ithreads)), ithreads, ismem, s>>>(
      d, e, static_cast<int>(l), evals, tn, scratch, piv, y, smem_ok ? ithreads : 0);
  backxform_kernel<<<gblocks, 32 * warps_per_block, 0, s>>>(refl, h, static_cast<int>(l), y, evecs);
  // refinement: scratch holds AZ, S, R, E; y receives Z E
  double* az = scratch;
  double* sm = az + l * l;
  double* rm = sm + l * l;
  double* em = rm + l * l;
  const int li = static_cast<int>(l);
  dim3 gg(static_cast<unsigned>(ceil_div(l, 64)), static_cast<unsigned>(ceil_div(l, 64)));
  dgemm_small<false><<<gg, 256, 0, s>>>(a, evecs, az, li);
  dgemm_small<true><<<gg, 256, 0, s>>>(evecs, az, sm, li);
  dgemm_small<true><<<gg, 256, 0, s>>>(evecs, evecs, rm, li);
  const unsigned eg = static_cast<unsigned>(ceil_div(l * l, 256));
  oa_correction_kernel<<<eg, 256, 0, s>>>(rm, sm, li, tn, em);
  dgemm_small<false><<<gg, 256, 0, s>>>(evecs, em, y, li);
  add_kernel<<<eg, 256, 0, s>>>(evecs, y, li * li);
}

}  // namespace lpca
