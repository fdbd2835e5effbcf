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
#include <cooperative_groups.h>
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

// 1 / x to within an ulp or two: the MUFU seed and two Newton steps (a quarter
// of the dependent latency of IEEE division, which dominates these recurrences).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double t = fma(-x, r, 1.0);
  r = fma(r, t, r);
  t = fma(-x, r, 1.0);
  return fma(r, t, r);
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

// Register-resident variant for l <= 32 CL. Warps 0-7 hold A: warp w owns rows
// w + 8 ra (ra < RW = 4 CL, cyclic so the active rows stay balanced over the
// warps as the corner shrinks) and lane L columns [CL L, CL L + CL); a step
// on the active i x i corner issues work only for active rows (the fp64 pipe,
// 2 warp-instructions per clock per SM, bounds the update). Warp 8 builds the
// reflectors one step ahead: during step i it takes row i - 1 as it was before
// the step (published by its owner), applies step i's rank-2 update to it on
// the fly by the same expression as the owners' register update, and forms
// reflector i - 1 while the owners update their rows, so the reflector's
// latency chain (two warp sums, a square root, reciprocals) is off the
// critical path. u, p, K partials go through double-buffered shared vectors;
// every warp forms K in the same order, so q = p - K u is bitwise the same
// everywhere and the update of (r, c) and (c, r) adds the same two products:
// A stays exactly symmetric. e, h and the reflectors stay in shared memory
// until the end. Two barriers per step.
constexpr int kTriRowWarps = 16;
constexpr int kTriBlkThreads = 32 * (kTriRowWarps + 1);

// Sum each of N per-lane values over the warp; lane L ends with the total of
// row idx (returned), lanes differing only in the low 5 - log2(N) bits agree.
template <int N>
__device__ __forceinline__ double reduce_scatter(double (&v)[N], int lane, int& idx) {
  idx = 0;
  int mask = 16;
#pragma unroll
  for (int hsz = N / 2; hsz >= 1; hsz /= 2) {
    const bool upper = (lane & mask) != 0;
#pragma unroll
    for (int j = 0; j < hsz; ++j) {
      const double send = upper ? v[j] : v[j + hsz];
      const double keep = upper ? v[j + hsz] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
    }
    if (upper) idx += hsz;
    mask >>= 1;
  }
  double t = v[0];
  for (; mask >= 1; mask >>= 1) t += __shfl_xor_sync(0xffffffffu, t, mask);
  return t;
}

#ifdef LPCA_TRI_PROF  // per-warp phase timing of tridiag_reg_kernel (tools/tri_prof.cu)
__device__ long long g_tri_prof[17][8];
#define TRI_PROF(k)                 \
  do {                              \
    const long long t_ = clock64(); \
    prof_acc[k] += t_ - prof_t;     \
    prof_t = t_;                    \
  } while (0)
#else
#define TRI_PROF(k) \
  do {              \
  } while (0)
#endif

template <int CL>
__global__ void __launch_bounds__(kTriBlkThreads) tridiag_reg_kernel(const double* __restrict__ a, int l,
                                                                     double* __restrict__ refl, double* d, double* e,
                                                                     double* h, double* norm_out, int* status,
                                                                     double* gap) {
  constexpr int NW = kTriRowWarps, W = 32 * CL, RW = W / NW, G = RW < 4 ? RW : 4;
  __shared__ double us[2][W];
  __shared__ double ps[2][W];
  __shared__ double rowb[W];
  __shared__ double hs[2];
  __shared__ int skip[2];
  __shared__ double kpart[2][NW];
  __shared__ double es[W];
  __shared__ double hsv[W];
  __shared__ double red[66];
  extern __shared__ double astage[];  // a, staged with coalesced loads; then the reflectors
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const bool builder = w == NW;
  const int c0 = CL * lane;
  for (int idx = tid; idx < l * l; idx += kTriBlkThreads) astage[idx] = a[idx];
  __syncthreads();
  double A[RW][CL];
  double fro = 0.0, asym = 0.0;
#pragma unroll
  for (int ra = 0; ra < RW; ++ra)
#pragma unroll
    for (int cb = 0; cb < CL; ++cb) {
      const int r = w + NW * ra, c = c0 + cb;
      double v = 0.0;
      if (!builder && r < l && c < l) {
        const double vrc = astage[c * l + r], vcr = astage[r * l + c];
        fro += vrc * vrc;
        asym = fmax(asym, fabs(vrc - vcr));
        v = r <= c ? vrc : vcr;  // exact symmetry from the upper triangle (tridiag_eigh.cpp:189-191)
      }
      A[ra][cb] = v;
    }
  fro = block_sum(fro, red);
  asym = block_max(asym, red);
  if (asym > 1e-10 * sqrt(fro)) {
    if (tid == 0) {
      status[0] = 2;
      gap[0] = asym;
    }
    return;
  }
  // the owner of row `row` copies it to rowb (visible after the next barrier)
  auto publish = [&](int row) {
    if (!builder && row % NW == w) {
#pragma unroll
      for (int ra = 0; ra < RW; ++ra)
        if (w + NW * ra == row) {
#pragma unroll
          for (int cb = 0; cb < CL; ++cb) rowb[c0 + cb] = A[ra][cb];
        }
    }
  };
  // builder: reflector ri from rowb (+ the pending update when upd) into the
  // (ri & 1) buffers
  auto build = [&](int ri, bool upd, double kk, const double* u, const double* p) {
    const int bb = ri & 1;
    double x[CL];
    if (upd) {
      const double ur = u[ri];
      const double qr = __dsub_rn(p[ri], __dmul_rn(kk, ur));
#pragma unroll
      for (int cb = 0; cb < CL; ++cb) {
        const double ucb = u[c0 + cb];
        const double qcb = __dsub_rn(p[c0 + cb], __dmul_rn(kk, ucb));
        x[cb] = __dsub_rn(rowb[c0 + cb], __dadd_rn(__dmul_rn(ur, qcb), __dmul_rn(qr, ucb)));
      }
    } else {
#pragma unroll
      for (int cb = 0; cb < CL; ++cb) x[cb] = rowb[c0 + cb];
    }
    double xl = 0.0;  // element ri - 1
#pragma unroll
    for (int cb = 0; cb < CL; ++cb)
      if (c0 + cb == ri - 1) xl = x[cb];
    xl = __shfl_sync(0xffffffffu, xl, (ri - 1) / CL);
    if (ri == 1) {
      if (lane == 0) {
        es[1] = xl;
        hsv[1] = 0.0;
        skip[bb] = 1;
      }
      return;
    }
    double pa = 0.0, ps2 = 0.0;
#pragma unroll
    for (int cb = 0; cb < CL; ++cb) {
      if (c0 + cb >= ri) x[cb] = 0.0;
      pa += fabs(x[cb]);
      ps2 += x[cb] * x[cb];
    }
    pa = warp_sum(pa);
    ps2 = warp_sum(ps2);
    if (pa == 0.0) {
      if (lane == 0) {
        es[ri] = 0.0;
        hsv[ri] = 0.0;
        skip[bb] = 1;
      }
      return;
    }
    const double inv = fast_rcp(pa);
    const double sigma = ps2 * inv * inv;
    const double f = xl * inv;
    const double g = f >= 0.0 ? -sqrt(sigma) : sqrt(sigma);
    const double hh = sigma - f * g;
#pragma unroll
    for (int cb = 0; cb < CL; ++cb) {
      const int c = c0 + cb;
      const double uv = c < ri - 1 ? x[cb] * inv : (c == ri - 1 ? f - g : 0.0);
      us[bb][c] = uv;
      if (c < ri) astage[ri * l + c] = uv;  // reflector ri (refl layout), for the back-transformation
    }
    if (lane == 0) {
      es[ri] = pa * g;
      hsv[ri] = hh;
      hs[bb] = fast_rcp(hh);
      skip[bb] = 0;
    }
  };
  __syncthreads();  // astage is free for the reflectors
  // The builder and the row warps run separate loops (the builder never holds
  // A, so neither path pays for the other's registers), meeting at the same
  // sequence of named barriers: one after the first publish, two per step.
  auto step_barrier = [] { asm volatile("bar.sync 1, %0;" ::"r"(kTriBlkThreads) : "memory"); };
  if (builder) {
    step_barrier();
    build(l - 1, false, 0.0, nullptr, nullptr);
    for (int i = l - 1; i >= 1; --i) {
      const int buf = i & 1;
      step_barrier();  // reflector i is ready
      const bool upd = !skip[buf];
      step_barrier();  // p, K partials and row i - 1 are ready
      if (i - 1 >= 1) {
        double kk = 0.0;
        if (upd) {
          double ksum = 0.0;
#pragma unroll
          for (int q = 0; q < NW; ++q) ksum += kpart[buf][q];
          kk = ksum * (0.5 * hs[buf] * hs[buf]);
        }
        build(i - 1, upd, kk, us[buf], ps[buf]);
      }
    }
  } else {
    publish(l - 1);
    step_barrier();
#ifdef LPCA_TRI_PROF
    long long prof_acc[8] = {};
    long long prof_t = clock64();
#endif
    for (int i = l - 1; i >= 1; --i) {
      const int buf = i & 1;
      const double* u = us[buf];
      double* p = ps[buf];
      step_barrier();  // reflector i is ready
      const bool upd = !skip[buf];
#ifdef LPCA_TRI_PROF
      if (skip[buf] == 12345) prof_t = 0;
#endif
      TRI_PROF(0);
      if (i - 1 >= 1) publish(i - 1);  // for the builder, as it is before this step's update
      // active rows w + NW ra < i come in groups of G register rows, one warp-
      // uniform branch per group; rows past i inside a group see u = p = 0, so
      // their update is an exact no-op
      const int ng = ((i - w + NW - 1) / NW + G - 1) / G;  // active row groups
      double uc[CL];
      double hinv = 0.0;
      if (upd) {
        hinv = hs[buf];
#pragma unroll
        for (int cb = 0; cb < CL; ++cb) uc[cb] = u[c0 + cb];
        double acc[RW];
        double uau = 0.0;  // this thread's share of u^T A u (K = u^T A u / 2 h^2)
#pragma unroll
        for (int g = 0; g < RW / G; ++g) {
          if (g < ng) {
#pragma unroll
            for (int q = 0; q < G; ++q) {
              const int ra = G * g + q;
              acc[ra] = 0.0;
#pragma unroll
              for (int cb = 0; cb < CL; ++cb) acc[ra] = fma(A[ra][cb], uc[cb], acc[ra]);
              uau = fma(u[w + NW * ra], acc[ra], uau);
            }
          } else {
#pragma unroll
            for (int q = 0; q < G; ++q) acc[G * g + q] = 0.0;
          }
        }
        int idx;
        const double sum = reduce_scatter<RW>(acc, lane, idx);
        uau = warp_sum(uau);
        if ((lane & (32 / RW - 1)) == 0) p[w + NW * idx] = w + NW * idx < i ? sum * hinv : 0.0;
        if (lane == 0) kpart[buf][w] = uau;
      }
      TRI_PROF(1);
      step_barrier();  // p, K partials and row i - 1 are ready
#ifdef LPCA_TRI_PROF
      if (kpart[buf][0] == 12345.5) prof_t = 0;
#endif
      TRI_PROF(2);
      if (upd) {
        double ksum = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) ksum += kpart[buf][q];
        const double kk = ksum * (0.5 * hinv * hinv);
        double qc[CL];
#pragma unroll
        for (int cb = 0; cb < CL; ++cb) qc[cb] = __dsub_rn(p[c0 + cb], __dmul_rn(kk, uc[cb]));
#pragma unroll
        for (int g = 0; g < RW / G; ++g) {
          if (g >= ng) break;
          double ur[G], qr[G];
#pragma unroll
          for (int q = 0; q < G; ++q) {
            ur[q] = u[w + NW * (G * g + q)];
            qr[q] = __dsub_rn(p[w + NW * (G * g + q)], __dmul_rn(kk, ur[q]));
          }
#pragma unroll
          for (int q = 0; q < G; ++q)
#pragma unroll
            for (int cb = 0; cb < CL; ++cb)
              A[G * g + q][cb] =
                  __dsub_rn(A[G * g + q][cb], __dadd_rn(__dmul_rn(ur[q], qc[cb]), __dmul_rn(qr[q], uc[cb])));
        }
      }
#ifdef LPCA_TRI_PROF
      if (A[0][0] == 12345.5) prof_t = 0;
#endif
      TRI_PROF(3);
    }
#ifdef LPCA_TRI_PROF
    if (lane == 0)
      for (int k = 0; k < 8; ++k) g_tri_prof[w][k] = prof_acc[k];
#endif
#pragma unroll
    for (int ra = 0; ra < RW; ++ra)
#pragma unroll
      for (int cb = 0; cb < CL; ++cb)
        if (w + NW * ra == c0 + cb && w + NW * ra < l) d[w + NW * ra] = A[ra][cb];
  }
  if (tid == 0) es[0] = 0.0;
  __syncthreads();
  // reflector i occupies refl[i l + c], c < i (the strictly upper part of astage)
  for (int idx = tid; idx < l * l; idx += kTriBlkThreads)
    if (idx % l < idx / l) refl[idx] = astage[idx];
  for (int k = tid; k < l; k += kTriBlkThreads) {
    e[k] = es[k];
    h[k] = k >= 1 ? hsv[k] : 0.0;
  }
  __syncthreads();
  double tn = 0.0;
  for (int k = tid; k < l; k += kTriBlkThreads) {
    const double ek = k > 0 ? fabs(es[k]) : 0.0, ek1 = k + 1 < l ? fabs(es[k + 1]) : 0.0;
    tn = fmax(tn, fabs(d[k]) + ek + ek1);
  }
  tn = block_max(tn, red);
  if (tid == 0) {
    norm_out[0] = tn;
    status[0] = 0;
    gap[0] = 0.0;
  }
}

// Multi-CTA variant for l > 128 (one cooperative grid, grid-wide syncs): CTA q
// of C holds rows q + C a (cyclic, so every CTA keeps work as the corner
// shrinks) in shared memory. Per step two grid syncs: the owner of row i builds
// reflector i from its row and publishes u, h (global, double-buffered by step
// parity) -> every CTA forms p = A u / h for its rows and a u^T p partial ->
// every CTA sums the partials in the same order, so K and q = p - K u are
// bitwise equal everywhere and the rank-2 update keeps A exactly symmetric; the
// owner of row i - 1 then builds the next reflector right after its update.
constexpr int kCoopThreads = 256, kCoopBatch = 8;

struct CoopWork {
  double* u;      // [2][l] reflectors by step parity
  double* p;      // [2][l]
  double* kpart;  // [2][C]
  double* fpart;  // [C] Frobenius / asymmetry partials
  double* apart;  // [C]
  double* hsv;    // [2] 1/h by parity; [2] skip flags as doubles at hsv + 2
};

// kCluster: the C CTAs form one thread-block cluster (C <= 16), meet at the
// hardware cluster barrier instead of a grid-wide sync, and exchange u, p, the
// K partials and 1/h through distributed shared memory: each value is stored
// into every CTA's copy before the barrier (st.shared::cluster), so after it
// all reads are local shared memory instead of L2 round trips (two per step;
// l = 220: 1.20 -> 0.90 ms; pulling each value after the barrier instead:
// 0.96 ms). The matvec and the rank-2 update load a lane's elements of a row
// before using them (the stores may alias, so the compiler cannot hoist).
// Same arithmetic in the same order: bitwise the same as the grid variant.
template <bool kCluster>
__global__ void __launch_bounds__(kCoopThreads) tridiag_coop_kernel(const double* __restrict__ a, int l,
                                                                    double* __restrict__ refl, double* d, double* e,
                                                                    double* h, double* norm_out, int* status,
                                                                    double* gap, CoopWork wk) {
  namespace cg = cooperative_groups;
  struct Sync {
    __device__ void sync() const {
      if (kCluster) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      } else {
        cg::this_grid().sync();
      }
    }
  } grid;
  extern __shared__ double rows_s[];  // [R][l], local row a = global row q + C a
  __shared__ double red[66];
  const int C = gridDim.x, q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int R = (l + C - 1) / C;
  // the exchanged vectors: this CTA's copies (cluster) or the global ones
  double* const xs = rows_s + static_cast<size_t>(R) * l;  // cluster: [2l u][2l p][2C kpart][4 hsv]
  double* const u_all = kCluster ? xs : wk.u;
  double* const p_all = kCluster ? xs + 2 * l : wk.p;
  double* const kp_all = kCluster ? xs + 4 * l : wk.kpart;
  double* const hsv = kCluster ? xs + 4 * l + 2 * C : wk.hsv;
  // store v at local address `at` of every CTA (cluster) / at the global one
  auto publish = [&](double* at, double v) {
    if (kCluster) {
      cg::cluster_group cl = cg::this_cluster();
      for (int t = 0; t < C; ++t) *cl.map_shared_rank(at, t) = v;
    } else {
      *at = v;
    }
  };
  // load (exact symmetry from the upper triangle, tridiag_eigh.cpp:189-191)
  double fro = 0.0, asym = 0.0;
  for (int idx = tid; idx < R * l; idx += kCoopThreads) {
    const int ra = idx / l, c = idx % l, r = q + C * ra;
    double v = 0.0;
    if (r < l) {
      const double vrc = a[static_cast<size_t>(c) * l + r], vcr = a[static_cast<size_t>(r) * l + c];
      fro += vrc * vrc;
      asym = fmax(asym, fabs(vrc - vcr));
      v = r <= c ? vrc : vcr;
    }
    rows_s[idx] = v;
  }
  fro = block_sum(fro, red);
  asym = block_max(asym, red);
  if (tid == 0) {
    wk.fpart[q] = fro;
    wk.apart[q] = asym;
  }
  grid.sync();
  {
    double f = 0.0, am = 0.0;
    for (int c = 0; c < C; ++c) {
      f += wk.fpart[c];
      am = fmax(am, wk.apart[c]);
    }
    if (am > 1e-10 * sqrt(f)) {
      if (q == 0 && tid == 0) {
        status[0] = 2;
        gap[0] = am;
      }
      return;  // grid-uniform
    }
  }
  // owner of row ri builds reflector ri from its (updated) shared-memory row
  auto build = [&](int ri) {
    const int bb = ri & 1;
    const double* row = rows_s + static_cast<size_t>(ri / C) * l;
    double* u = u_all + static_cast<size_t>(bb) * l;
    if (ri == 1) {
      if (tid == 0) {
        e[1] = row[0];
        h[1] = 0.0;
        publish(&hsv[2 + bb], 1.0);
      }
      return;
    }
    double pa = 0.0, ps2 = 0.0;
    for (int c = tid; c < ri; c += kCoopThreads) {
      pa += fabs(row[c]);
      ps2 += row[c] * row[c];
    }
    block_sum2(pa, ps2, red);
    if (pa == 0.0) {
      if (tid == 0) {
        e[ri] = 0.0;
        h[ri] = 0.0;
        publish(&hsv[2 + bb], 1.0);
      }
      return;
    }
    const double inv = fast_rcp(pa);
    const double sigma = ps2 * inv * inv;
    const double f = row[ri - 1] * inv;
    const double g = f >= 0.0 ? -sqrt(sigma) : sqrt(sigma);
    const double hh = sigma - f * g;
    for (int c = tid; c < ri; c += kCoopThreads) {
      const double uv = c < ri - 1 ? row[c] * inv : f - g;
      publish(&u[c], uv);
      refl[static_cast<size_t>(ri) * l + c] = uv;  // for the back-transformation
    }
    if (tid == 0) {
      e[ri] = pa * g;
      h[ri] = hh;
      publish(&hsv[bb], fast_rcp(hh));
      publish(&hsv[2 + bb], 0.0);
    }
  };
  if (q == (l - 1) % C) build(l - 1);
  for (int i = l - 1; i >= 1; --i) {
    const int bb = i & 1;
    grid.sync();  // reflector i published
    const bool skip = hsv[2 + bb] != 0.0;
    const double* u = u_all + static_cast<size_t>(bb) * l;
    double* p = p_all + static_cast<size_t>(bb) * l;
    const int nra = i > q ? (i - q + C - 1) / C : 0;  // own active rows q + C a < i
    if (!skip) {
      const double hinv = hsv[bb];
      double pu = 0.0;
      for (int ra = w; ra < nra; ra += kCoopThreads / 32) {  // warp per row
        const double* row = rows_s + static_cast<size_t>(ra) * l;
        double acc = 0.0;
        for (int c0 = lane; c0 < i; c0 += 32 * kCoopBatch) {
          double rv[kCoopBatch], uv[kCoopBatch];
#pragma unroll
          for (int t = 0; t < kCoopBatch; ++t) {
            const int c = c0 + 32 * t;
            rv[t] = c < i ? row[c] : 0.0;
            uv[t] = c < i ? u[c] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < kCoopBatch; ++t)
            if (c0 + 32 * t < i) acc = fma(rv[t], uv[t], acc);
        }
        acc = warp_sum(acc) * hinv;
        const int r = q + C * ra;
        if (lane == 0) publish(&p[r], acc);
        pu = fma(u[r], acc, pu);  // lane-uniform value: counted once below
      }
      if (lane != 0) pu = 0.0;
      pu = block_sum(pu, red);
      if (tid == 0) publish(&kp_all[bb * C + q], pu);
    }
    grid.sync();  // p and the K partials published
    if (!skip) {
      double ksum = 0.0;
      for (int c = 0; c < C; ++c) ksum += kp_all[bb * C + c];
      const double kk = ksum * (0.5 * hsv[bb]);
      for (int ra = w; ra < nra; ra += kCoopThreads / 32) {  // warp per row, lanes along it
        const int r = q + C * ra;
        const double ur = u[r], qr = __dsub_rn(p[r], __dmul_rn(kk, ur));
        double* xrow = rows_s + static_cast<size_t>(ra) * l;
        for (int c0 = lane; c0 < i; c0 += 32 * kCoopBatch) {
          double uv[kCoopBatch], pv[kCoopBatch], xv[kCoopBatch];
#pragma unroll
          for (int t = 0; t < kCoopBatch; ++t) {
            const int c = c0 + 32 * t;
            uv[t] = c < i ? u[c] : 0.0;
            pv[t] = c < i ? p[c] : 0.0;
            xv[t] = c < i ? xrow[c] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < kCoopBatch; ++t) {
            const int c = c0 + 32 * t;
            const double qc = __dsub_rn(pv[t], __dmul_rn(kk, uv[t]));
            if (c < i) xrow[c] = __dsub_rn(xv[t], __dadd_rn(__dmul_rn(ur, qc), __dmul_rn(qr, uv[t])));
          }
        }
      }
      __syncthreads();
    }
    if (i - 1 >= 1 && q == (i - 1) % C) build(i - 1);
  }
  for (int ra = tid; ra < R; ra += kCoopThreads) {
    const int r = q + C * ra;
    if (r < l) d[r] = rows_s[static_cast<size_t>(ra) * l + r];
  }
  if (q == 0 && tid == 0) e[0] = 0.0;
  grid.sync();
  if (q == 0) {
    double tn = 0.0;
    for (int k = tid; k < l; k += kCoopThreads) {
      const double ek = k > 0 ? fabs(e[k]) : 0.0, ek1 = k + 1 < l ? fabs(e[k + 1]) : 0.0;
      tn = fmax(tn, fabs(d[k]) + ek + ek1);
    }
    tn = block_max(tn, red);
    if (tid == 0) {
      norm_out[0] = tn;
      status[0] = 0;
      gap[0] = 0.0;
    }
  }
}

// ---- 2. multisection ---------------------------------------------------------------------
// Number of eigenvalues of T strictly below x (Sturm sequence of T - x I);
// ee[i] = e[i]^2, |q| kept >= pivmin (normal), so the reciprocal is finite.
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ ee, int l,
                                           double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < l; ++i) {
    q = (d[i] - x) - ee[i] * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// One CTA of kBisThreads per eigenvalue j (descending; ascending index
// t = l-1-j): every thread probes one point per round, so a round narrows the
// bracket kBisThreads + 1 fold (7 bits) instead of bisection's 2; d and e^2 are
// staged in shared memory.
constexpr int kBisThreads = 128;

__device__ __forceinline__ double probe_point(double lo, double w, int k) {
  return __fma_rn(w, static_cast<double>(k + 1) / (kBisThreads + 1), lo);
}

__global__ void __launch_bounds__(kBisThreads) bisect_kernel(const double* __restrict__ d,
                                                             const double* __restrict__ e, int l,
                                                             const double* __restrict__ tnorm, double* evals) {
  extern __shared__ double bsm[];
  double* ds = bsm;
  double* ee = bsm + l;
  __shared__ double red[2 * (kBisThreads / 32) + 2];
  __shared__ unsigned long long bal[kBisThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int j = blockIdx.x;
  double lo = DBL_MAX, hi = -DBL_MAX, emax2 = 0.0;
  for (int i = tid; i < l; i += kBisThreads) {
    const double ei = i > 0 ? fabs(e[i]) : 0.0, ei1 = i + 1 < l ? fabs(e[i + 1]) : 0.0;
    ds[i] = d[i];
    ee[i] = ei * ei;
    lo = fmin(lo, d[i] - ei - ei1);
    hi = fmax(hi, d[i] + ei + ei1);
    emax2 = fmax(emax2, ei * ei);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
  }
  if (lane == 0) {
    red[wid] = lo;
    red[kBisThreads / 32 + wid] = hi;
    bal[wid] = __double_as_longlong(emax2);
  }
  __syncthreads();
  for (int w = 0; w < kBisThreads / 32; ++w) {
    lo = fmin(lo, red[w]);
    hi = fmax(hi, red[kBisThreads / 32 + w]);
    emax2 = fmax(emax2, __longlong_as_double(bal[w]));
  }
  __syncthreads();
  const double tn = tnorm[0];
  const double pivmin = DBL_MIN * fmax(1.0, emax2);
  const double abstol = 2.0 * DBL_EPSILON * fmax(tn, DBL_MIN);
  lo -= abstol;
  hi += abstol;
  const int t = l - 1 - j;
  for (int round = 0; round < 40; ++round) {
    const double w = hi - lo;
    if (w <= abstol + 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) break;
    const double x = probe_point(lo, w, tid);
    const int c = (x > lo && x < hi) ? sturm_count(ds, ee, l, x, pivmin) : (x <= lo ? 0 : l);
    // the first probe whose count exceeds t bounds the eigenvalue from above
    const unsigned above = __ballot_sync(0xffffffffu, c > t);
    if (lane == 0) bal[wid] = above;
    __syncthreads();
    int k = kBisThreads;  // first probe index above, over the whole CTA
    for (int q = 0; q < kBisThreads / 32; ++q)
      if (bal[q]) {
        k = q * 32 + __ffs(static_cast<unsigned>(bal[q])) - 1;
        break;
      }
    __syncthreads();
    // probe points are recomputed (the same expression) rather than exchanged
    const double nhi = k < kBisThreads ? probe_point(lo, w, k) : hi;
    const double nlo = k > 0 ? probe_point(lo, w, k - 1) : lo;
    lo = nlo;
    hi = nhi;
  }
  if (tid == 0) evals[j] = 0.5 * (lo + hi);
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

// T - lam I = P L U by pivoted LU (the dgttrf recurrences), factored once per
// shift; the running pivot row lives in registers. Fields: DL (multipliers),
// D (1 / pivot), DU, DU2.
__device__ void tri_factor(const double* __restrict__ d, const double* __restrict__ e, int l, double lam, double tiny,
                           const Scr& s, unsigned char* piv) {
  enum { DL = 0, D = 1, DU = 2, DU2 = 3 };
  double dcur = d[0] - lam, ducur = l > 1 ? e[1] : 0.0;
  for (int i = 0; i + 1 < l; ++i) {
    const double dli = e[i + 1];
    double dnext = d[i + 1] - lam, dunext = i + 2 < l ? e[i + 2] : 0.0;
    if (fabs(dcur) >= fabs(dli)) {
      const double pd = fabs(dcur) < tiny ? (dcur < 0 ? -tiny : tiny) : dcur;
      const double rp = fast_rcp(pd);
      const double fact = dli * rp;
      s.at(D, i) = rp;
      s.at(DL, i) = fact;
      s.at(DU, i) = ducur;
      s.at(DU2, i) = 0.0;
      dnext -= fact * ducur;
      piv[i] = 0;
    } else {
      const double rl = fabs(dli) >= DBL_MIN ? fast_rcp(dli) : 1.0 / dli;  // (the seed flushes subnormals)
      const double fact = dcur * rl;
      s.at(D, i) = rl;
      s.at(DL, i) = fact;
      s.at(DU, i) = dnext;
      s.at(DU2, i) = dunext;
      dnext = ducur - fact * dnext;
      dunext = -fact * dunext;
      piv[i] = 1;
    }
    dcur = dnext;
    ducur = dunext;
  }
  if (fabs(dcur) < tiny) dcur = dcur < 0 ? -tiny : tiny;
  s.at(D, l - 1) = fast_rcp(dcur);
}

// b <- (T - lam I)^{-1} b with the factors of tri_factor (dgttrs), b in field 4.
__device__ void tri_apply(int l, const Scr& s, const unsigned char* piv) {
  enum { DL = 0, D = 1, DU = 2, DU2 = 3, B = 4 };
  double bi = s.at(B, 0);
  for (int i = 0; i + 1 < l; ++i) {
    double bn = s.at(B, i + 1);
    if (!piv[i]) {
      bn -= s.at(DL, i) * bi;
      s.at(B, i) = bi;
    } else {
      s.at(B, i) = bn;
      bn = bi - s.at(DL, i) * bn;
    }
    bi = bn;
  }
  double x1 = bi * s.at(D, l - 1), x2 = 0.0;
  s.at(B, l - 1) = x1;
  if (l > 1) {
    x2 = x1;
    x1 = (s.at(B, l - 2) - s.at(DU, l - 2) * x2) * s.at(D, l - 2);
    s.at(B, l - 2) = x1;
  }
  for (int i = l - 3; i >= 0; --i) {
    const double x = (s.at(B, i) - s.at(DU, i) * x1 - s.at(DU2, i) * x2) * s.at(D, i);
    s.at(B, i) = x;
    x2 = x1;
    x1 = x;
  }
}

__device__ __forceinline__ bool same_cluster(double a, double b, double tn) {
  const double scale = fmax(fabs(a), fabs(b));
  return fabs(a - b) <= 1e-3 * scale || scale <= 1e-13 * tn;
}

// Y (row-major, Y[i * l + j] = component i of eigenvector j of T). One warp
// per eigenvalue: lane 0 runs the serial LU recurrences (its scratch in shared
// memory), the warp does the vector-wide passes (start vector, Gram-Schmidt,
// scaling, store). Only cluster leaders work; they walk their cluster in order.
__global__ void invit_kernel(const double* __restrict__ d, const double* __restrict__ e, int l,
                             const double* __restrict__ evals, const double* __restrict__ tnorm,
                             double* __restrict__ y, int wpb) {
  extern __shared__ double sh_scr[];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int j = blockIdx.x * wpb + wid;
  if (j >= l) return;
  const double tn = tnorm[0] > 0.0 ? tnorm[0] : 1.0;  // zero matrix: any orthonormal basis
  if (j > 0 && same_cluster(evals[j - 1], evals[j], tn)) return;
  int end = j + 1;
  while (end < l && same_cluster(evals[end - 1], evals[end], tn)) ++end;
  double* base = sh_scr + static_cast<size_t>(wid) * 5 * l;
  const Scr s{base, l, 0, 1};
  double* b = base + static_cast<size_t>(4) * l;
  unsigned char* piv = reinterpret_cast<unsigned char*>(sh_scr + static_cast<size_t>(5) * l * wpb) +
                       static_cast<size_t>(wid) * l;
  const double tiny = DBL_EPSILON * tn;
  double prev_shift = 0.0;
  for (int jj = j; jj < end; ++jj) {
    double lam = evals[jj];
    if (jj > j && lam >= prev_shift - 10.0 * DBL_EPSILON * fmax(fabs(lam), tn * 1e-6))
      lam = prev_shift - 10.0 * DBL_EPSILON * fmax(fabs(lam), tn * 1e-6);  // separate equal shifts
    prev_shift = lam;
    for (int i = lane; i < l; i += 32) b[i] = hash_uniform(static_cast<unsigned>(jj), static_cast<unsigned>(i));
    if (lane == 0) tri_factor(d, e, l, lam, tiny, s, piv);
    __syncwarp();
    for (int it = 0; it < 3; ++it) {
      if (lane == 0) tri_apply(l, s, piv);
      __syncwarp();
      // modified Gram-Schmidt against the cluster's earlier vectors, twice: a
      // cluster at the roundoff floor (rank-deficient G) leaves a remainder far
      // smaller than the iterate, and one pass loses orthogonality to cancellation
      for (int pass = 0; pass < (jj > j ? 2 : 0); ++pass)
        for (int pj = j; pj < jj; ++pj) {
          double dot = 0.0;
          for (int i = lane; i < l; i += 32) dot += y[static_cast<size_t>(i) * l + pj] * b[i];
          dot = warp_sum(dot);
          for (int i = lane; i < l; i += 32) b[i] -= dot * y[static_cast<size_t>(i) * l + pj];
          __syncwarp();
        }
      double mx = 0.0;
      for (int i = lane; i < l; i += 32) mx = fmax(mx, fabs(b[i]));
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (mx == 0.0) {
        for (int i = lane; i < l; i += 32)
          b[i] = hash_uniform(static_cast<unsigned>(jj) + 7919u, static_cast<unsigned>(i));
        __syncwarp();
        continue;
      }
      const double rmx = 1.0 / mx;
      double nrm = 0.0;
      for (int i = lane; i < l; i += 32) {
        const double v = b[i] * rmx;
        nrm += v * v;
      }
      const double sc = rmx / sqrt(warp_sum(nrm));
      for (int i = lane; i < l; i += 32) b[i] *= sc;
      __syncwarp();
    }
    for (int i = lane; i < l; i += 32) y[static_cast<size_t>(i) * l + jj] = b[i];
    __syncwarp();
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

// Same sweep with the eigenvector in registers (lane owns rows lane + 32 b) and
// the reflectors (and 1 / h) staged in shared memory when they fit: each
// reflector costs a dot, one warp sum and an axpy with no global round trip.
template <int RB>
__global__ void backxform_reg_kernel(const double* __restrict__ refl, const double* __restrict__ h, int l,
                                     const double* __restrict__ y, double* __restrict__ z, int refl_smem) {
  extern __shared__ double sref[];
  const double* R = refl;
  double* hinv = sref + (refl_smem ? static_cast<size_t>(l) * l : 0);
  if (refl_smem) {
    for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) sref[idx] = refl[idx];
    R = sref;
  }
  for (int i = threadIdx.x; i < l; i += blockDim.x) hinv[i] = h[i] != 0.0 ? 1.0 / h[i] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x % 32;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (j >= l) return;
  double zr[RB];
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    const int k = lane + 32 * b;
    zr[b] = k < l ? y[static_cast<size_t>(k) * l + j] : 0.0;
  }
  for (int i = 1; i < l; ++i) {
    const double hi = hinv[i];
    if (hi == 0.0) continue;
    const double* u = R + static_cast<size_t>(i) * l;
    double uk[RB];
    double dot = 0.0;
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int k = lane + 32 * b;
      uk[b] = k < i ? u[k] : 0.0;
      if (k < i) dot = fma(uk[b], zr[b], dot);
    }
    dot = warp_sum(dot) * hi;
#pragma unroll
    for (int b = 0; b < RB; ++b)
      if (lane + 32 * b < i) zr[b] = fma(-dot, uk[b], zr[b]);
  }
  double* zj = z + static_cast<size_t>(j) * l;
#pragma unroll
  for (int b = 0; b < RB; ++b)
    if (lane + 32 * b < l) zj[lane + 32 * b] = zr[b];
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
__global__ void __launch_bounds__(256) dgemm_small(const double* __restrict__ a, const double* __restrict__ b0,
                                                   double* __restrict__ c0, const double* __restrict__ b1,
                                                   double* __restrict__ c1, const double* __restrict__ addc, int l) {
  // C (l x l) = [addc +] op(A) B, all column-major l x l; op(A) = A^T when
  // kTransA; blockIdx.z picks (B, C) = (b0, c0) or (b1, c1). 16 x 16 tiles, one
  // output per thread with two partial sums: at these sizes the load latency
  // and the FMA chain, not the fp64 rate, bound the kernel, so it wants many
  // small CTAs (49 at l = 110).
  constexpr int T = 16, BK = 64;
  __shared__ double As[BK][T + 1];  // As[kk][ii] = op(A)(i0 + ii, k0 + kk)
  __shared__ double Bs[T][BK + 1];  // Bs[jj][kk] = B(k0 + kk, j0 + jj)
  const double* __restrict__ b = blockIdx.z ? b1 : b0;
  double* __restrict__ c = blockIdx.z ? c1 : c0;
  const int tid = threadIdx.x, tx = tid % T, ty = tid / T;
  const int i0 = blockIdx.x * T, j0 = blockIdx.y * T;
  double acc0 = 0.0, acc1 = 0.0;
  for (int k0 = 0; k0 < l; k0 += BK) {
#pragma unroll
    for (int q = 0; q < (T * BK) / 256; ++q) {
      const int idx = tid + 256 * q;
      if (kTransA) {  // A^T(gi, gk) = a[gi * l + gk]: coalesced over k
        const int kk = idx % BK, ii = idx / BK, gi = i0 + ii, gk = k0 + kk;
        As[kk][ii] = (gi < l && gk < l) ? a[static_cast<size_t>(gi) * l + gk] : 0.0;
      } else {  // A(gi, gk) = a[gk * l + gi]: coalesced over i
        const int ii = idx % T, kk = idx / T, gi = i0 + ii, gk = k0 + kk;
        As[kk][ii] = (gi < l && gk < l) ? a[static_cast<size_t>(gk) * l + gi] : 0.0;
      }
      const int kk = idx % BK, jj = idx / BK, gj = j0 + jj, gk = k0 + kk;
      Bs[jj][kk] = (gj < l && gk < l) ? b[static_cast<size_t>(gj) * l + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll 16
    for (int kk = 0; kk < BK; kk += 2) {
      acc0 = fma(As[kk][tx], Bs[ty][kk], acc0);
      acc1 = fma(As[kk + 1][tx], Bs[ty][kk + 1], acc1);
    }
    __syncthreads();
  }
  const int gi = i0 + tx, gj = j0 + ty;
  if (gi < l && gj < l) {
    const double v = acc0 + acc1;
    c[static_cast<size_t>(gj) * l + gi] = addc ? addc[static_cast<size_t>(gj) * l + gi] + v : v;
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
  // S carries absolute roundoff ~eps ||A||: below an absolute gap of 1e-8 ||A||
  // the separated formula would amplify it past 1e-8, so such pairs are only
  // orthogonalised (their vectors are determined no better than that anyway)
  const bool cluster = fabs(ltj - lti) <= fmax(1e-3 * scale, 1e-8 * tn) || scale <= 1e-13 * tn;
  e[idx] = cluster ? 0.5 * rij : (sij + ltj * rij) / (ltj - lti);
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
  const std::size_t amat = static_cast<std::size_t>(l * l) * sizeof(double);
  const std::size_t vecs = static_cast<std::size_t>(3 * l) * sizeof(double);
  const int a_smem = amat + vecs <= 200 * 1024 ? 1 : 0;
  const std::size_t smem = (a_smem ? amat : 0) + vecs;
  const int li = static_cast<int>(l);
  if (l <= 32) {
    tridiag_reg_kernel<1><<<1, kTriBlkThreads, amat, s>>>(a, li, refl, d, e, h, tn, status, gap);
  } else if (l <= 64) {
    tridiag_reg_kernel<2><<<1, kTriBlkThreads, amat, s>>>(a, li, refl, d, e, h, tn, status, gap);
  } else if (l <= 128) {
    LPCA_CUDA(cudaFuncSetAttribute(tridiag_reg_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(amat)));
    tridiag_reg_kernel<4><<<1, kTriBlkThreads, amat, s>>>(a, li, refl, d, e, h, tn, status, gap);
  } else {
    // one cluster of up to 16 CTAs (hardware barrier) while the rows fit their
    // shared memory, else a cooperative grid of ~8 rows per CTA
    const std::size_t row_bytes = static_cast<std::size_t>(l) * sizeof(double);
    const bool cluster = static_cast<std::size_t>(ceil_div(l, 16)) * row_bytes <= 200 * 1024;
    int C = cluster ? static_cast<int>(ceil_div(l, ceil_div(l, 16))) : static_cast<int>(ceil_div(l, 8));
    C = cluster ? C : (C < 8 ? 8 : (C > 148 ? 148 : C));
    const std::size_t csm = static_cast<std::size_t>(ceil_div(l, C)) * row_bytes;
    if (csm <= 200 * 1024) {
      CoopWork wk;
      wk.u = scratch;  // the refinement's scratch is free during the tridiagonalisation
      wk.p = wk.u + 2 * l;
      wk.kpart = wk.p + 2 * l;
      wk.fpart = wk.kpart + 2 * C;
      wk.apart = wk.fpart + C;
      wk.hsv = wk.apart + C;
      if (cluster) {
        const std::size_t xsm = csm + static_cast<std::size_t>(4 * l + 2 * C + 4) * sizeof(double);  // + exchange
        LPCA_CUDA(cudaFuncSetAttribute(tridiag_coop_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(xsm)));
        LPCA_CUDA(cudaFuncSetAttribute(tridiag_coop_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(kCoopThreads);
        cfg.dynamicSmemBytes = xsm;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        LPCA_CUDA(cudaLaunchKernelEx(&cfg, tridiag_coop_kernel<true>, a, li, refl, d, e, h, tn, status, gap, wk));
      } else {
        LPCA_CUDA(cudaFuncSetAttribute(tridiag_coop_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(csm)));
        void* args[] = {&a, const_cast<int*>(&li), &refl, &d, &e, &h, &tn, &status, &gap, &wk};
        LPCA_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(tridiag_coop_kernel<false>), dim3(C),
                                              dim3(kCoopThreads), args, csm, s));
      }
    } else {
      LPCA_CUDA(cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      tridiag_kernel<<<1, kTriThreads, smem, s>>>(a, li, refl, a_smem, d, e, h, tn, status, gap);
    }
  }
  const int warps_per_block = 4;
  const unsigned gblocks = static_cast<unsigned>(ceil_div(l, warps_per_block));
  const std::size_t bis_smem = static_cast<std::size_t>(2 * l) * sizeof(double);
  if (bis_smem > 48 * 1024)
    LPCA_CUDA(cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bis_smem)));
  bisect_kernel<<<static_cast<unsigned>(l), kBisThreads, bis_smem, s>>>(d, e, li, tn, evals);
  int wpb = 4;  // warps per block: 5 l doubles + l pivot bytes of scratch each
  while (wpb > 1 && static_cast<std::size_t>(wpb) * 41 * l > 200 * 1024) wpb >>= 1;
  const std::size_t ismem = static_cast<std::size_t>(wpb) * 41 * l + 16;
  if (ismem > 227 * 1024) throw Error(kInternal, "eigh: inverse-iteration scratch exceeds shared memory");
  LPCA_CUDA(cudaFuncSetAttribute(invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ismem)));
  invit_kernel<<<static_cast<unsigned>(ceil_div(l, wpb)), 32 * wpb, ismem, s>>>(d, e, li, evals, tn, y, wpb);
  const int rsm = amat + static_cast<std::size_t>(l) * sizeof(double) <= 200 * 1024 ? 1 : 0;
  const std::size_t bsm = (rsm ? amat : 0) + static_cast<std::size_t>(l) * sizeof(double);
  if (l <= 128) {
    LPCA_CUDA(cudaFuncSetAttribute(backxform_reg_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bsm)));
    backxform_reg_kernel<4><<<static_cast<unsigned>(ceil_div(l, 8)), 256, bsm, s>>>(refl, h, li, y, evecs, rsm);
  } else if (l <= 512) {
    LPCA_CUDA(cudaFuncSetAttribute(backxform_reg_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bsm)));
    backxform_reg_kernel<16><<<static_cast<unsigned>(ceil_div(l, 8)), 256, bsm, s>>>(refl, h, li, y, evecs, rsm);
  } else {
    backxform_kernel<<<gblocks, 32 * warps_per_block, 0, s>>>(refl, h, li, y, evecs);
  }
  // refinement, two passes (the second squares what the first leaves in
  // pairs it could only orthogonalise): scratch holds AZ, S, R, E; Z ping-pongs
  // between evecs and y and ends in evecs
  double* az = scratch;
  double* sm = az + l * l;
  double* rm = sm + l * l;
  double* em = rm + l * l;
  const dim3 gg(static_cast<unsigned>(ceil_div(l, 16)), static_cast<unsigned>(ceil_div(l, 16)));
  const dim3 gg2(gg.x, gg.y, 2);
  const unsigned eg = static_cast<unsigned>(ceil_div(l * l, 256));
  for (int pass = 0; pass < 2; ++pass) {
    double* z = pass == 0 ? evecs : y;
    double* zn = pass == 0 ? y : evecs;
    dgemm_small<false><<<gg, 256, 0, s>>>(a, z, az, nullptr, nullptr, nullptr, li);
    dgemm_small<true><<<gg2, 256, 0, s>>>(z, az, sm, z, rm, nullptr, li);
    oa_correction_kernel<<<eg, 256, 0, s>>>(rm, sm, li, tn, em);
    dgemm_small<false><<<gg, 256, 0, s>>>(z, em, zn, nullptr, nullptr, z, li);
  }
}

}  // namespace lpca
