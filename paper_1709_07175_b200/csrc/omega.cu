// Projection generation, synthetic data and layout helpers.
#include <cuda_runtime.h>

#include <mutex>
#include <unordered_set>
#include <vector>

#include "kernels.cuh"
#include "rng.cuh"

namespace lpca {

namespace {

constexpr int kOmegaThreads = 256;
constexpr int kOmegaSeg = 128;                   // draws per lane per round
constexpr int kOmegaChunk = 32 * kOmegaSeg;      // draws per round (32 KB of smem)
constexpr int kJumps = 33;                       // T^(128 L), L = 0..31, and T^4096

// xoshiro256** is linear over GF(2) in its 256-bit state: advancing J draws is
// a fixed 256 x 256 bit matrix T^J. Column j of matrix k is T^J e_j (four
// 64-bit words, s0..s3). With them the 32 lanes of a warp start at draws
// 128 L of their column's stream and walk 128 draws each, instead of one lane
// walking all of them: the same raw sequence. Lane L makes one jump, T^(128 L)
// (its own matrix), and every further round one T^4096.
// Stored column-interleaved, g_jump[j][k][w]: for a fixed column j the 32
// lanes' matrices (k = lane) are contiguous, so each step of the product is
// one coalesced 1 KB read across the warp.
__device__ __align__(16) std::uint64_t g_jump[256][kJumps][4];

__device__ __forceinline__ void jump_state(int k, Xoshiro& x) {
  const std::uint64_t in[4] = {x.s0, x.s1, x.s2, x.s3};
  std::uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll 4
  for (int j = 0; j < 256; ++j) {
    const std::uint64_t bit = (in[j >> 6] >> (j & 63)) & 1ull;
    const std::uint64_t mask = 0ull - bit;
    const ulonglong2 lo = *reinterpret_cast<const ulonglong2*>(&g_jump[j][k][0]);
    const ulonglong2 hi = *reinterpret_cast<const ulonglong2*>(&g_jump[j][k][2]);
    o0 ^= lo.x & mask;
    o1 ^= lo.y & mask;
    o2 ^= hi.x & mask;
    o3 ^= hi.y & mask;
  }
  x.s0 = o0;
  x.s1 = o1;
  x.s2 = o2;
  x.s3 = o3;
}

// Raw draws [base, base + 4096) of `col`'s stream into raw[], round `round`
// (base = 4096 round): lane L of warp 0 jumps to draw base + 128 L.
__device__ __forceinline__ void omega_raw_round(Xoshiro& lane_state, int round, index_t n, std::uint64_t* raw) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    if (round > 0) jump_state(32, lane_state);  // +4096 from this lane's previous round start
    Xoshiro x = lane_state;
    const index_t base = static_cast<index_t>(round) * kOmegaChunk + lane * kOmegaSeg;
    for (int t = 0; t < kOmegaSeg && base + t < n; ++t) raw[lane * kOmegaSeg + t] = x.next();
  }
}

// Lane L's start state T^(128 L) s. The 32 lanes' matrices (256 KB, usually
// evicted from L2 by the X passes between fits) are streamed through shared
// memory by the whole CTA in 32-column chunks (coalesced 16 B loads), warp 0
// folding each chunk into its product. Call with all threads; lanes of warp 0
// get their state, other threads a dummy.
__device__ Xoshiro omega_lane_start(std::uint64_t seed, index_t col, std::uint64_t* stage) {
  constexpr int kCols = kOmegaChunk * 8 / (32 * 32);  // columns per chunk that fit the 32 KB stage
  Xoshiro x = column_stream(seed, static_cast<std::uint64_t>(col));
  const int lane = threadIdx.x & 31;
  const std::uint64_t in[4] = {x.s0, x.s1, x.s2, x.s3};
  std::uint64_t o[4] = {0, 0, 0, 0};
  for (int j0 = 0; j0 < 256; j0 += kCols) {
    // g_jump[j][k][w] for j in [j0, j0 + kCols), k < 32: one contiguous block
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(&g_jump[j0][0][0]);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(stage);
    for (int e = threadIdx.x; e < kCols * 32 * 2; e += kOmegaThreads) {
      const int jj = e / 64, rest = e % 64;  // 64 ulonglong2 per column (32 lanes x 2)
      dst[e] = src[jj * (kJumps * 2) + rest];
    }
    __syncthreads();
    if (threadIdx.x < 32) {
#pragma unroll 4
      for (int jj = 0; jj < kCols; ++jj) {
        const int j = j0 + jj;
        const std::uint64_t mask = 0ull - ((in[j >> 6] >> (j & 63)) & 1ull);
        const std::uint64_t* m = stage + (jj * 32 + lane) * 4;
#pragma unroll
        for (int w = 0; w < 4; ++w) o[w] ^= m[w] & mask;
      }
    }
    __syncthreads();
  }
  if (lane > 0) {
    x.s0 = o[0];
    x.s1 = o[1];
    x.s2 = o[2];
    x.s3 = o[3];
  }
  return x;
}

// One CTA per projection column (gen_gaussian runs one task per column,
// projection.cpp:71-84): warp 0 produces the column's raw 64-bit draws (32
// lanes at jumped stream positions), then the whole CTA maps them through
// normal_icdf and writes the column with coalesced stores.
__global__ void __launch_bounds__(kOmegaThreads) omega_gaussian_kernel(index_t n, std::uint64_t seed,
                                                                       double* out, index_t ld) {
  __shared__ std::uint64_t raw[kOmegaChunk];
  const index_t col = blockIdx.x;
  Xoshiro st = omega_lane_start(seed, col, raw);  // raw doubles as the jump-matrix stage
  double* dst = out + col * ld;
  for (index_t base = 0, round = 0; base < n; base += kOmegaChunk, ++round) {
    const int cnt = static_cast<int>(n - base < kOmegaChunk ? n - base : kOmegaChunk);
    omega_raw_round(st, static_cast<int>(round), n, raw);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += kOmegaThreads) dst[base + i] = normal_icdf(u64_to_uniform(raw[i]));
    __syncthreads();
  }
}

// gen_very_sparse (projection.cpp:86-126): one uniform per cell, u < d/2 -> +1,
// d/2 <= u < d -> -1, else 0. Dense {-1,0,+1} column, unscaled.
__global__ void __launch_bounds__(kOmegaThreads) omega_sparse_kernel(index_t n, double density,
                                                                     std::uint64_t seed, double* out,
                                                                     index_t ld) {
  __shared__ std::uint64_t raw[kOmegaChunk];
  const index_t col = blockIdx.x;
  Xoshiro st = omega_lane_start(seed, col, raw);  // raw doubles as the jump-matrix stage
  double* dst = out + col * ld;
  const double half = density / 2.0;
  for (index_t base = 0, round = 0; base < n; base += kOmegaChunk, ++round) {
    const int cnt = static_cast<int>(n - base < kOmegaChunk ? n - base : kOmegaChunk);
    omega_raw_round(st, static_cast<int>(round), n, raw);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += kOmegaThreads) {
      const double u = u64_to_uniform(raw[i]);
      dst[base + i] = u >= density ? 0.0 : (u < half ? 1.0 : -1.0);
    }
    __syncthreads();
  }
}

// Host: the jump matrices, computed once and uploaded to each device used.
void xoshiro_step(std::uint64_t (&s)[4]) {
  const std::uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

void ensure_jump_tables(cudaStream_t s) {
  static std::vector<std::uint64_t> host;  // [kJumps][256][4]
  static std::mutex mu;
  static std::unordered_set<int> ready;
  int dev = 0;
  LPCA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (ready.count(dev)) return;
  if (host.empty()) {
    host.assign(static_cast<std::size_t>(kJumps) * 256 * 4, 0);
    // T^(128 L) column by column, each from the previous L's by 128 more steps
    for (int j = 0; j < 256; ++j) {
      std::uint64_t st[4] = {0, 0, 0, 0};
      st[j >> 6] = 1ull << (j & 63);
      for (int L = 0; L < 32; ++L) {
        if (L > 0)
          for (int t = 0; t < kOmegaSeg; ++t) xoshiro_step(st);
        for (int w = 0; w < 4; ++w) host[(static_cast<std::size_t>(j) * kJumps + L) * 4 + w] = st[w];
      }
      for (int t = 0; t < kOmegaSeg; ++t) xoshiro_step(st);  // 32 * 128 = 4096
      for (int w = 0; w < 4; ++w) host[(static_cast<std::size_t>(j) * kJumps + 32) * 4 + w] = st[w];
    }
  }
  LPCA_CUDA(cudaMemcpyToSymbolAsync(g_jump, host.data(), host.size() * sizeof(std::uint64_t), 0,
                                    cudaMemcpyHostToDevice, s));
  LPCA_CUDA(cudaStreamSynchronize(s));  // host buffer is static; the sync keeps the first use simple
  ready.insert(dev);
}

// ---- synthetic low-rank data --------------------------------------------------
// G (rows x r, already scaled by sigma_t) and H (r x n) are materialised for one
// row batch; X tiles are then a K = r DFMA product with t ascending, plus the
// counter-based noise term, rounded once to the storage dtype.
__global__ void synth_factor_kernel(index_t row0, index_t rows, index_t r, index_t n,
                                    const double* sigma, std::uint64_t seed, double* gs, double* h,
                                    bool make_h) {
  const index_t tid = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x;
  const index_t stride = static_cast<index_t>(gridDim.x) * blockDim.x;
  const std::uint64_t seed_g = seed + 1001, seed_h = seed + 1002;
  for (index_t e = tid; e < rows * r; e += stride) {
    const index_t i = e / r, t = e % r;
    gs[e] = counter_normal(seed_g, static_cast<std::uint64_t>((row0 + i) * r + t)) * sigma[t];
  }
  if (make_h)
    for (index_t e = tid; e < r * n; e += stride)
      h[e] = counter_normal(seed_h, static_cast<std::uint64_t>(e));
}

template <typename TO>
__global__ void __launch_bounds__(256) synth_gemm_kernel(index_t row0, index_t rows, index_t n,
                                                         index_t r, const double* gs,
                                                         const double* h, double noise,
                                                         std::uint64_t seed, TO* x, index_t ldx,
                                                         index_t x_row_off) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ double As[BK][BM + 1];
  __shared__ double Bs[BK][BN];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const index_t i0 = static_cast<index_t>(blockIdx.y) * BM, j0 = static_cast<index_t>(blockIdx.x) * BN;
  double acc[4][4] = {};
  for (index_t t0 = 0; t0 < r; t0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      const int mi = e / BK, kk = e % BK;
      const index_t gi = i0 + mi, gt = t0 + kk;
      As[kk][mi] = (gi < rows && gt < r) ? gs[gi * r + gt] : 0.0;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      const int kk = e / BN, nj = e % BN;
      const index_t gt = t0 + kk, gj = j0 + nj;
      Bs[kk][nj] = (gt < r && gj < n) ? h[gt * n + gj] : 0.0;
    }
    __syncthreads();
    const int kmax = static_cast<int>(r - t0 < BK ? r - t0 : BK);
    for (int kk = 0; kk < kmax; ++kk)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(As[kk][ty * 4 + a], Bs[kk][tx * 4 + b], acc[a][b]);
    __syncthreads();
  }
  const std::uint64_t seed_e = seed + 1003;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const index_t gi = i0 + ty * 4 + a;
    if (gi >= rows) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const index_t gj = j0 + tx * 4 + b;
      if (gj >= n) continue;
      const double e = counter_normal(seed_e, static_cast<std::uint64_t>((row0 + gi) * n + gj));
      x[(x_row_off + gi) * ldx + gj] = static_cast<TO>(fma(noise, e, acc[a][b]));
    }
  }
}

__global__ void convert_kernel(const double* src, index_t lds, float* dst, index_t ldd,
                               index_t rows, index_t cols, double scale) {
  const index_t total = rows * cols;
  for (index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<index_t>(gridDim.x) * blockDim.x) {
    const index_t c = e / rows, i = e % rows;
    dst[c * ldd + i] = static_cast<float>(src[c * lds + i] * scale);
  }
}

__global__ void scale_kernel(const double* src, double* dst, index_t count, double inv) {
  for (index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<index_t>(gridDim.x) * blockDim.x)
    dst[e] = src[e] * inv;
}

__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

__global__ void split_w_kernel(const double* w, index_t ldw, index_t n, index_t wc, index_t wpad,
                               float* hi, float* lo, index_t ldd) {
  const index_t total = wpad * ldd;
  for (index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<index_t>(gridDim.x) * blockDim.x) {
    const index_t c = e / ldd, j = e % ldd;
    float h = 0.f, lw = 0.f;
    if (c < wc && j < n) {
      const double v = w[c * ldw + j];
      h = tf32_trunc(static_cast<float>(v));
      lw = tf32_trunc(static_cast<float>(v - static_cast<double>(h)));
    }
    hi[e] = h;
    lo[e] = lw;
  }
}

__global__ void split_rows_kernel(const float* src, index_t count, float* hi, float* lo) {
  for (index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; e < count;
       e += static_cast<index_t>(gridDim.x) * blockDim.x) {
    const float v = src[e];
    const float h = tf32_trunc(v);
    hi[e] = h;
    lo[e] = tf32_trunc(v - h);
  }
}

// 32 x 32 tiles through shared memory: coalesced reads of src rows, coalesced
// writes of the transposed planes.
__global__ void split_transpose_kernel(const float* src, index_t m, index_t cols, index_t lds, float* hi,
                                       float* lo, index_t ldt) {
  __shared__ float tile[32][33];
  const index_t r0 = static_cast<index_t>(blockIdx.x) * 32, c0 = static_cast<index_t>(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const index_t r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < m && c < cols) ? src[r * lds + c] : 0.f;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const index_t c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < m) {
      const float v = tile[threadIdx.x][k];
      const float h = tf32_trunc(v);
      hi[c * ldt + r] = h;
      lo[c * ldt + r] = tf32_trunc(v - h);
    }
  }
}

template <typename TO>
__global__ void csc_to_dense_kernel(index_t n, const std::int64_t* col_ptr,
                                    const std::int64_t* row_idx, const double* vals, TO* x,
                                    index_t ldx) {
  for (index_t j = blockIdx.x; j < n; j += gridDim.x)
    for (std::int64_t p = col_ptr[j] + threadIdx.x; p < col_ptr[j + 1]; p += blockDim.x)
      x[row_idx[p] * ldx + j] = static_cast<TO>(vals[p]);
}

template <typename T>
__global__ void transpose_kernel(const T* src, index_t lds, index_t rows, index_t cols, T* dst,
                                 index_t ldd) {
  __shared__ T tile[32][33];
  const index_t r0 = static_cast<index_t>(blockIdx.x) * 32, c0 = static_cast<index_t>(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const index_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[c * lds + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const index_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) dst[r * ldd + c] = tile[threadIdx.x][k];
  }
}

__global__ void widen_kernel(const float* src, index_t lds, index_t m, index_t n, double* dst) {
  const index_t total = m * n;
  for (index_t e = blockIdx.x * static_cast<index_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<index_t>(gridDim.x) * blockDim.x)
    dst[e] = static_cast<double>(src[(e / n) * lds + e % n]);
}

int grid_for(index_t work, int threads) {
  index_t g = ceil_div(work, threads);
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

void launch_omega_gaussian(cudaStream_t s, index_t n, index_t l, std::uint64_t seed, double* out,
                           index_t ld) {
  if (l <= 0 || n <= 0) return;
  ensure_jump_tables(s);
  omega_gaussian_kernel<<<static_cast<unsigned>(l), kOmegaThreads, 0, s>>>(n, seed, out, ld);
}

void launch_omega_very_sparse(cudaStream_t s, index_t n, index_t l, double density,
                              std::uint64_t seed, double* out, index_t ld) {
  if (l <= 0 || n <= 0) return;
  ensure_jump_tables(s);
  omega_sparse_kernel<<<static_cast<unsigned>(l), kOmegaThreads, 0, s>>>(n, density, seed, out, ld);
}

void launch_synth_lowrank(cudaStream_t s, index_t row0, index_t m, index_t n, index_t r,
                          const double* sigma_dev, double noise, std::uint64_t seed, int dtype,
                          void* x, index_t ldx, double* scratch, index_t scratch_elems) {
  double* h = scratch;
  double* gs = scratch + r * n;
  index_t batch = (scratch_elems - r * n) / r;
  if (batch > m) batch = m;
  if (batch < 64) throw Error(kInternal, "synth: scratch too small");
  bool make_h = true;
  for (index_t b0 = 0; b0 < m; b0 += batch) {
    const index_t rows = m - b0 < batch ? m - b0 : batch;
    synth_factor_kernel<<<grid_for(rows * r + (make_h ? r * n : 0), 256), 256, 0, s>>>(
        row0 + b0, rows, r, n, sigma_dev, seed, gs, h, make_h);
    make_h = false;
    dim3 grid(static_cast<unsigned>(ceil_div(n, 64)), static_cast<unsigned>(ceil_div(rows, 64)));
    if (dtype == 4)
      synth_gemm_kernel<float><<<grid, 256, 0, s>>>(row0 + b0, rows, n, r, gs, h, noise, seed,
                                                    static_cast<float*>(x), ldx, b0);
    else
      synth_gemm_kernel<double><<<grid, 256, 0, s>>>(row0 + b0, rows, n, r, gs, h, noise, seed,
                                                     static_cast<double*>(x), ldx, b0);
  }
}

void launch_convert_f64_to_f32(cudaStream_t s, const double* src, index_t lds, float* dst,
                               index_t ldd, index_t rows, index_t cols, double scale) {
  convert_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(src, lds, dst, ldd, rows, cols, scale);
}

void launch_scale_f64(cudaStream_t s, const double* src, double* dst, index_t count, double inv) {
  scale_kernel<<<grid_for(count, 256), 256, 0, s>>>(src, dst, count, inv);
}

// One CTA per W column: the column's max |w| sets a power-of-two scale
// 2^(14 - floor(log2 max)) (as tc_pair.cuh's pow2_scale_for), then
// hi = fp16_rn(w s), lo = fp16_rn(w s - hi).
__global__ void split_f16_w_kernel(const double* __restrict__ w, index_t ldw, index_t n, index_t wc,
                                   __half* __restrict__ hi, __half* __restrict__ lo, index_t ldd,
                                   float* __restrict__ winv, int* __restrict__ lo_nz) {
  const index_t c = blockIdx.x;
  __shared__ float red[32];
  float mx = 0.0f;
  if (c < wc)
    for (index_t j = threadIdx.x; j < n; j += blockDim.x) mx = fmaxf(mx, fabsf(static_cast<float>(w[c * ldw + j])));
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) red[0] = mx;
  }
  __syncthreads();
  mx = red[0];
  float sc = 1.0f;
  if (mx > 0.0f && !isinf(mx)) {
    int e = 14 - ilogbf(mx);
    e = e > 126 ? 126 : (e < -126 ? -126 : e);
    sc = ldexpf(1.0f, e);
  }
  if (threadIdx.x == 0) winv[c] = 1.0f / sc;
  int any_lo = 0;
  for (index_t j = threadIdx.x; j < ldd; j += blockDim.x) {
    const float y = (c < wc && j < n) ? static_cast<float>(w[c * ldw + j] * static_cast<double>(sc)) : 0.0f;
    const __half h = __float2half_rn(y);
    const __half l = __float2half_rn(y - __half2float(h));
    hi[c * ldd + j] = h;
    lo[c * ldd + j] = l;
    any_lo |= __half_as_ushort(l) & 0x7fff;
  }
  if (__syncthreads_or(any_lo) && threadIdx.x == 0 && lo_nz) atomicOr(lo_nz, 1);
}

void launch_split_f16_w(cudaStream_t s, const double* w, index_t ldw, index_t n, index_t wc, index_t wpad,
                        __half* hi, __half* lo, index_t ldd, float* winv, int* lo_nz) {
  if (wpad <= 0) return;
  if (lo_nz) LPCA_CUDA(cudaMemsetAsync(lo_nz, 0, sizeof(int), s));
  split_f16_w_kernel<<<static_cast<unsigned>(wpad), 256, 0, s>>>(w, ldw, n, wc, hi, lo, ldd, winv, lo_nz);
}

void launch_split_tf32_w(cudaStream_t s, const double* w, index_t ldw, index_t n, index_t wc,
                         index_t wpad, float* hi, float* lo, index_t ldd) {
  split_w_kernel<<<grid_for(wpad * ldd, 256), 256, 0, s>>>(w, ldw, n, wc, wpad, hi, lo, ldd);
}

void launch_split_tf32_rows(cudaStream_t s, const float* src, index_t m, index_t ld, float* hi,
                            float* lo) {
  split_rows_kernel<<<grid_for(m * ld, 256), 256, 0, s>>>(src, m * ld, hi, lo);
}

void launch_split_tf32_transpose(cudaStream_t s, const float* src, index_t m, index_t cols, index_t lds,
                                 float* hi, float* lo, index_t ldt) {
  if (m <= 0 || cols <= 0) return;
  dim3 grid(static_cast<unsigned>(ceil_div(m, 32)), static_cast<unsigned>(ceil_div(cols, 32)));
  split_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(src, m, cols, lds, hi, lo, ldt);
}

void launch_csc_to_dense(cudaStream_t s, index_t m, index_t n, const std::int64_t* col_ptr,
                         const std::int64_t* row_idx, const double* vals, int dtype, void* x,
                         index_t ldx) {
  (void)m;
  const unsigned g = static_cast<unsigned>(n < 148 * 8 ? n : 148 * 8);
  if (n <= 0) return;
  if (dtype == 4)
    csc_to_dense_kernel<float><<<g, 128, 0, s>>>(n, col_ptr, row_idx, vals, static_cast<float*>(x), ldx);
  else
    csc_to_dense_kernel<double><<<g, 128, 0, s>>>(n, col_ptr, row_idx, vals, static_cast<double*>(x), ldx);
}

void launch_transpose(cudaStream_t s, int dtype, const void* src, index_t lds, index_t rows,
                      index_t cols, void* dst, index_t ldd) {
  dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(ceil_div(cols, 32)));
  dim3 block(32, 8);
  if (dtype == 4)
    transpose_kernel<float><<<grid, block, 0, s>>>(static_cast<const float*>(src), lds, rows, cols,
                                                   static_cast<float*>(dst), ldd);
  else
    transpose_kernel<double><<<grid, block, 0, s>>>(static_cast<const double*>(src), lds, rows,
                                                    cols, static_cast<double*>(dst), ldd);
}

void launch_widen_f32(cudaStream_t s, const float* src, index_t lds, index_t m, index_t n, double* dst) {
  widen_kernel<<<grid_for(m * n, 256), 256, 0, s>>>(src, lds, m, n, dst);
}

void launch_zero(cudaStream_t s, void* p, std::size_t bytes) {
  LPCA_CUDA(cudaMemsetAsync(p, 0, bytes, s));
}

}  // namespace lpca
