// The sketch U = X Omega for a very sparse Omega (gen_very_sparse,
// proj/core/src/projection.cpp:86-126: entries in {-1, 0, +1}, about n l d of
// them) as a gather: U[i, c] = sum over j in nz(c) of Omega[j, c] X[i, j]
// (spmm with a CSC Omega, proj/core/src/kernels.cpp:49-68, visits the same
// (j, c) pairs). One read of X and no multiplies: HBM-bound, where the dense
// tensor-core pass over the same X is tensor-bound (BASELINE configs[3]:
// n = 16,384, l = 300, d = 1/128).
//
// Omega is first turned into per-(K chunk of 256 columns, Omega column) lists
// of its nonzeros, each entry the byte offset of X[row 0, j] in the kernel's
// tile pair: the chunk of X, and its negation (so an entry's sign is its
// address), lists padded to even length with the tile's zero column. The
// gather kernel is persistent over tiles of 64 rows (fp32) or 32 rows (fp64);
// each chunk is loaded with coalesced 16-byte loads into registers one chunk
// ahead and stored into rows padded by one element, so the 32 lanes of a warp
// — one row each — read one column j from 32 different banks. Warp w keeps the
// sums of its contiguous block of columns for its rows in registers across the
// chunks, walking each column's entries two at a time: every U entry is summed
// left to right in ascending j, as spmm does (fp64: the reference's bits).
// max|X| comes from the staged registers.
//
// Measured (profiles/r02_c4_sparse_sketch.txt): about 1.6 TB/s, a quarter of
// HBM; the walk is latency-bound (short lists per chunk and column, exposed
// load latency at each chunk's barrier). fp32 X takes the row gather below
// (long rows) or the dense 2-SM pass (short rows), so the fit runs this kernel
// for fp64 X (lpca.cu sparse_omega_mode).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace lpca {
namespace {

constexpr int kRows = 32;               // rows per tile = lanes
constexpr int kWarps = 16;              // column groups
constexpr int kThreadsSO = 32 * kWarps;

template <typename T>
__host__ __device__ constexpr int chunk_cols() {
  return 256;  // 64 (fp32) or 128 (fp64) 16-byte vectors per row
}
template <typename T>
__host__ __device__ constexpr int rows_per_lane() {
  return sizeof(T) == 4 ? 2 : 1;  // a chunk of the tile is 4096 16-byte vectors either way
}

// counts[t * l + c] = nonzeros of Omega column c in rows [t kc, (t + 1) kc)
__global__ void omega_chunk_count_kernel(const double* __restrict__ omega, index_t n, index_t l, int kc, int nchunks,
                                         int* __restrict__ counts) {
  const index_t e = static_cast<index_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<index_t>(nchunks) * l) return;
  const index_t t = e / l, c = e % l;
  const index_t j0 = t * kc, j1 = j0 + kc < n ? j0 + kc : n;
  int cnt = 0;
  for (index_t j = j0; j < j1; ++j) cnt += omega[c * n + j] != 0.0;
  counts[e] = (cnt + 1) & ~1;  // segments padded to pairs (padding: the zero column kc)
}

// Exclusive scan of `count` ints in one CTA (ptr has count + 1 entries).
__global__ void scan_kernel(const int* __restrict__ counts, index_t count, int* __restrict__ ptr) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (index_t base = 0; base < count; base += blockDim.x) {
    const index_t i = base + threadIdx.x;
    int v = i < count ? counts[i] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int w = lane < static_cast<int>(blockDim.x >> 5) ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int before = carry + (wid > 0 ? warp_sums[wid - 1] : 0);
    if (i < count) ptr[i] = before + incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) ptr[count] = carry;
}

// entries[ptr[t l + c] ...]: the byte offset of X[row 0, j] in the gather
// kernel's tile pair (+X, then -X at element offset neg_off), j - t kc
// ascending; then a padding entry (the zero column kc) up to an even count
__global__ void omega_chunk_fill_kernel(const double* __restrict__ omega, index_t n, index_t l, int kc, int nchunks,
                                        const int* __restrict__ ptr, std::uint32_t* __restrict__ ent, int neg_off,
                                        int esize) {
  const index_t e = static_cast<index_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<index_t>(nchunks) * l) return;
  const index_t t = e / l, c = e % l;
  const index_t j0 = t * kc, j1 = j0 + kc < n ? j0 + kc : n;
  int p = ptr[e];
  const int end = ptr[e + 1];
  for (index_t j = j0; j < j1; ++j) {
    const double w = omega[c * n + j];
    if (w != 0.0) ent[p++] = static_cast<std::uint32_t>(((j - j0) + (w < 0.0 ? neg_off : 0)) * esize);
  }
  while (p < end) ent[p++] = static_cast<std::uint32_t>(kc * esize);
}

// Element q of a 16-byte vector (4 floats or 2 doubles), without taking addresses.
template <typename T, int q>
__device__ __forceinline__ T vec_elem(const float4& v) {
  if constexpr (sizeof(T) == 4) {
    return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
  } else {
    return q == 0 ? __hiloint2double(__float_as_int(v.y), __float_as_int(v.x))
                  : __hiloint2double(__float_as_int(v.w), __float_as_int(v.z));
  }
}

template <typename T>
__device__ __forceinline__ float4 vec_make(const T* e) {
  if constexpr (sizeof(T) == 4) {
    return make_float4(e[0], e[1], e[2], e[3]);
  } else {
    return make_float4(__int_as_float(__double2loint(e[0])), __int_as_float(__double2hiint(e[0])),
                       __int_as_float(__double2loint(e[1])), __int_as_float(__double2hiint(e[1])));
  }
}

// Loads one chunk of the tile (32 RPL rows x 256 columns = 4096 16-byte
// vectors) into registers, 8 vectors per thread. Pass k of thread (warp w,
// lane L) takes virtual row 4 k + L / 8 and virtual vector 8 w + L % 8 of a
// 32 x 128 grid (a warp instruction reads 4 x 128 contiguous bytes); a virtual
// row is RPL consecutive rows of X. The stores into rows padded by one element
// are conflict-free for fp64 and at most 2-way for fp32.
template <typename T>
__device__ __forceinline__ void chunk_coords(int k, int warp, int lane, int& row, int& vec) {
  constexpr int VPR = chunk_cols<T>() * static_cast<int>(sizeof(T)) / 16;  // vectors per row
  const int vr = 4 * k + lane / 8, vv = 8 * warp + lane % 8;
  row = vr * (128 / VPR) + vv / VPR;
  vec = vv % VPR;
}

template <typename T>
__device__ __forceinline__ void load_chunk(const T* __restrict__ x, index_t m, index_t n, index_t ldx, index_t r0,
                                           index_t j0, int warp, int lane, float4 (&v)[8]) {
  constexpr int V = 16 / sizeof(T);
  const bool aligned = ((ldx * sizeof(T)) & 15) == 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int row, vec;
    chunk_coords<T>(k, warp, lane, row, vec);
    const index_t r = r0 + row, j = j0 + static_cast<index_t>(vec) * V;
    if (r < m && j + V <= n && aligned) {
      v[k] = __ldg(reinterpret_cast<const float4*>(x + r * ldx + j));
    } else {  // ragged tail, rows past m, or unaligned rows: element by element
      T e[V];
#pragma unroll
      for (int q = 0; q < V; ++q) e[q] = (r < m && j + q < n) ? x[r * ldx + j + q] : T(0);
      v[k] = vec_make<T>(e);
    }
  }
}

constexpr int kEntCap = 16384;  // a chunk's staged entries (more: read from L2)

// Warp w owns columns [w cpw, (w + 1) cpw) and keeps their sums for its rows in
// registers across the chunks (MC >= cpw). Per chunk and column it walks the
// column's entries four at a time (one 16-byte broadcast load), each adding
// +-X[row, j] with an FFMA by +-1: every U entry is summed left to right in
// ascending j, as spmm does, padding entries adding the zero column.
template <typename T, int RPL, int MC>
__global__ void __launch_bounds__(kThreadsSO, 1)
    sparse_sketch_kernel(const T* __restrict__ x, index_t m, index_t n, index_t ldx, const int* __restrict__ ptr,
                         const std::uint32_t* __restrict__ ent, int l, int nchunks, T* __restrict__ u, index_t ldu,
                         std::uint32_t* xmax) {
  constexpr int kc = chunk_cols<T>();
  constexpr int stride = kc + 1;  // column kc stays zero; lanes (= rows) reading one column hit distinct banks
  constexpr int V = 16 / sizeof(T);
  constexpr int rows = kRows * RPL;
  constexpr int neg_off = rows * stride;  // -X follows +X: a list entry's sign is its address
  extern __shared__ __align__(16) unsigned char so_smem[];
  T* xs = reinterpret_cast<T*>(so_smem);                                              // [2][rows][stride]
  int* sptr = reinterpret_cast<int*>(xs + ((2 * rows * stride + 1) & ~1));             // [l + 1]
  std::uint32_t* sent = reinterpret_cast<std::uint32_t*>(sptr + ((kWarps * MC + 1 + 3) & ~3));  // [kEntCap]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cpw = (l + kWarps - 1) / kWarps;
  const int cw0 = min(l, warp * cpw), ncol = min(l, cw0 + cpw) - cw0;
  const index_t tiles = (m + rows - 1) / rows;
  float amax = 0.0f;
  float4 stage[8];
  for (int r = threadIdx.x; r < 2 * rows; r += kThreadsSO) xs[r * stride + kc] = T(0);

  for (index_t tile_i = blockIdx.x; tile_i < tiles; tile_i += gridDim.x) {
    const index_t r0 = tile_i * rows;
    T acc[MC][RPL];
#pragma unroll
    for (int i = 0; i < MC; ++i)
#pragma unroll
      for (int h = 0; h < RPL; ++h) acc[i][h] = T(0);
    load_chunk<T>(x, m, n, ldx, r0, 0, warp, lane, stage);
    for (int t = 0; t < nchunks; ++t) {
      __syncthreads();  // the previous chunk's readers are done
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        int row, vec;
        chunk_coords<T>(k, warp, lane, row, vec);
        T* dst = xs + row * stride + vec * V;
        const T a0 = vec_elem<T, 0>(stage[k]), a1 = vec_elem<T, 1>(stage[k]);
        dst[0] = a0;
        dst[1] = a1;
        dst[neg_off] = -a0;
        dst[neg_off + 1] = -a1;
        amax = fmaxf(amax, fmaxf(fabsf(static_cast<float>(a0)), fabsf(static_cast<float>(a1))));
        if constexpr (V == 4) {
          const T a2 = vec_elem<T, 2>(stage[k]), a3 = vec_elem<T, 3>(stage[k]);
          dst[2] = a2;
          dst[3] = a3;
          dst[neg_off + 2] = -a2;
          dst[neg_off + 3] = -a3;
          amax = fmaxf(amax, fmaxf(fabsf(static_cast<float>(a2)), fabsf(static_cast<float>(a3))));
        }
      }
      const int* pt = ptr + static_cast<index_t>(t) * l;
      const int e0 = __ldg(pt), e1 = __ldg(pt + l);
      const bool staged = e1 - e0 <= kEntCap;
      for (int c = threadIdx.x; c <= l; c += kThreadsSO) sptr[c] = __ldg(pt + c) - e0;
      if (staged)
        for (int q = 2 * threadIdx.x; q < e1 - e0; q += 2 * kThreadsSO)
          *reinterpret_cast<uint2*>(sent + q) = __ldg(reinterpret_cast<const uint2*>(ent + e0 + q));
      __syncthreads();
      if (t + 1 < nchunks)  // the next chunk is in flight while this one is reduced
        load_chunk<T>(x, m, n, ldx, r0, static_cast<index_t>(t + 1) * kc, warp, lane, stage);
      const unsigned char* xrow = reinterpret_cast<const unsigned char*>(xs + lane * stride);
      auto walk = [&](const std::uint32_t* es) {
#pragma unroll
        for (int i = 0; i < MC; ++i) {
          if (i < ncol) {
            const int q1 = sptr[cw0 + i + 1];
            for (int q = sptr[cw0 + i]; q < q1; q += 2) {
              const uint2 w = *reinterpret_cast<const uint2*>(es + q);
              const unsigned char* a0 = xrow + w.x;
              const unsigned char* a1 = xrow + w.y;
#pragma unroll
              for (int h = 0; h < RPL; ++h) {
                acc[i][h] += *reinterpret_cast<const T*>(a0 + h * kRows * stride * sizeof(T));
                acc[i][h] += *reinterpret_cast<const T*>(a1 + h * kRows * stride * sizeof(T));
              }
            }
          }
        }
      };
      if (staged)  // the launcher sizes the staging area for the density; L2 otherwise
        walk(sent);
      else
        walk(ent + e0);
    }
#pragma unroll
    for (int h = 0; h < RPL; ++h) {
      const index_t r = r0 + lane + kRows * h;
      if (r < m) {
        T* urow = u + r * ldu;
#pragma unroll
        for (int i = 0; i < MC; ++i)
          if (i < ncol) urow[cw0 + i] = acc[i][h];
        for (int c = kWarps * cpw + warp; c < ldu; c += kWarps) urow[c] = T(0);  // padding columns
        if (warp == kWarps - 1)
          for (int c = l; c < kWarps * cpw && c < ldu; ++c) urow[c] = T(0);
      }
    }
  }
  if (xmax) {
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) atomicMax(xmax, __float_as_uint(amax));
  }
}

// U^T fp16 hi/lo planes scaled per (column, kUScaleRows-row block) from a plain
// row-major fp32 U: the layout the X^T U pair kernel reads (the same rule as
// the X W pass epilogue, tc_pair.cuh: s = 2^(14 - floor(log2 max|U|)) per
// column and block, hi = fp16(u s), lo = fp16(u s - hi), inverse scale kept).
// One CTA per kUScaleRows-row block and 32-column group; thread = row.
__global__ void __launch_bounds__(kUScaleRows) u_planes_f16_kernel(const float* __restrict__ u, index_t m, index_t ld,
                                                           index_t npad, __half* __restrict__ hi,
                                                           __half* __restrict__ lo, index_t ldt,
                                                           float* __restrict__ uinv) {
  constexpr int kW = static_cast<int>(kUScaleRows) / 32;
  __shared__ float red[kW][32];
  __shared__ float scl[32];
  const index_t blk = blockIdx.x;
  const index_t row = blk * kUScaleRows + threadIdx.x;
  const index_t c0 = static_cast<index_t>(blockIdx.y) * 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = (row < m && c0 + k < npad) ? u[row * ld + c0 + k] : 0.0f;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    float a = fabsf(v[k]);
    for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0) red[wid][k] = a;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float a = 0.0f;
    for (int w = 0; w < kW; ++w) a = fmaxf(a, red[w][threadIdx.x]);
    float s = 1.0f;
    if (a > 0.0f && !isinf(a)) {
      int e = static_cast<int>((__float_as_uint(a) >> 23) & 0xffu) - 127;
      e = e < -126 ? -126 : e;
      int t = 14 - e;
      t = t > 126 ? 126 : (t < -126 ? -126 : t);
      s = __uint_as_float(static_cast<uint32_t>(t + 127) << 23);
    }
    scl[threadIdx.x] = s;
    if (c0 + threadIdx.x < npad) uinv[blk * npad + c0 + threadIdx.x] = __frcp_rn(s);
  }
  __syncthreads();
  if (row < m) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (c0 + k >= npad) break;
      const float y = v[k] * scl[k];
      const __half h = __float2half_rn(y);
      hi[(c0 + k) * ldt + row] = h;
      lo[(c0 + k) * ldt + row] = __float2half_rn(y - __half2float(h));
    }
  }
}


// ---------------------------------------------------------------------------
// Row gather for fp32 X (sparse_sketch_rows_kernel): lanes are Omega columns.
// Each CTA streams whole rows of X into a ring of shared-memory slots with
// 1-D bulk copies (TMA engine, no register staging), and every warp sums its
// 32 columns' entries of the row: lane c adds +-x[j] for the j of column c.
// The order of each lane's entries is a precomputed schedule (host edge
// colouring, build_row_schedule): at every step the 32 lanes of a warp read 32
// different banks, so each step is one shared-memory wavefront. A step's idle
// lanes read zeros from a free bank. Entries are 16 bits (word index | sign <<
// 15), two per register, the whole row's schedule held in registers. fp32 sums
// in the schedule's order (fp32 X only: the fp64 path keeps the reference's
// ascending order, sparse_sketch_kernel).

// cols[c * cap + i]: the i-th nonzero of Omega column c, j | (sign << 31), j
// ascending; cnt[c] = the column's nonzeros (entries past cap are dropped).
__global__ void omega_col_lists_kernel(const double* __restrict__ omega, index_t n, index_t l, int cap,
                                       int* __restrict__ cnt, std::uint32_t* __restrict__ cols) {
  const index_t c = static_cast<index_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (c >= l) return;
  int k = 0;
  for (index_t j0 = 0; j0 < n; j0 += 32) {
    const index_t j = j0 + lane;
    const double w = j < n ? omega[c * n + j] : 0.0;
    const unsigned nz = __ballot_sync(0xffffffffu, w != 0.0);
    const int pos = k + __popc(nz & ((1u << lane) - 1u));
    if (w != 0.0 && pos < cap) cols[c * cap + pos] = static_cast<std::uint32_t>(j) | (w < 0.0 ? 0x80000000u : 0u);
    k += __popc(nz);
  }
  if (lane == 0) cnt[c] = k;
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// The schedule takes SMAX / 2 registers per thread, which bounds the CTA: P = 2
// splits each row's entries by j into two halves run by separate warps (twice
// the warps to hide the loads' latency; the halves' sums meet in shared memory).
constexpr int rows_max_threads(int smax, int splits) {
  return splits == 2 ? (smax <= 64 ? 768 : 640) : (smax > 128 ? 320 : 512);
}

template <int SMAX, int P>
__global__ void __launch_bounds__(rows_max_threads(SMAX, P), 1)
    sparse_sketch_rows_kernel(const float* __restrict__ x, index_t m, int n, index_t ldx,
                              const std::uint32_t* __restrict__ sched, int steps, int slot_floats, int ring, int l,
                              float* __restrict__ u, index_t ldu, std::uint32_t* xmax) {
  extern __shared__ __align__(128) unsigned char rows_smem[];
  float* slots = reinterpret_cast<float*>(rows_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(slots + static_cast<size_t>(ring) * slot_floats);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wps = static_cast<int>(blockDim.x >> 5) / P;  // column warps per split
  const int part = warp / wps;                             // which half of j this warp sums
  const int col = (warp % wps) * 32 + lane;
  float* red = reinterpret_cast<float*>(full + 4);  // [2][wps * 32]: the second half's sums, by row parity
  // the whole row's schedule of this lane, two 16-bit entries per register
  std::uint32_t e[SMAX / 2];
#pragma unroll
  for (int i = 0; i < SMAX / 2; ++i) e[i] = __ldg(sched + (static_cast<size_t>(warp) * (SMAX / 2) + i) * 32 + lane);
  for (int r = 0; r < ring; ++r)
    for (int j = n + threadIdx.x; j < slot_floats; j += blockDim.x) slots[static_cast<size_t>(r) * slot_floats + j] = 0.f;
  if (threadIdx.x == 0) {
    for (int r = 0; r < ring; ++r) tc::mbar_init(&full[r], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  const uint32_t row_bytes = static_cast<uint32_t>(n) * 4u;
  if (threadIdx.x == 0)
    for (int r = 0; r < ring; ++r) {
      const index_t row = blockIdx.x + static_cast<index_t>(r) * gridDim.x;
      if (row < m) {
        tc::mbar_expect_tx(&full[r], row_bytes);
        bulk_load(slots + static_cast<size_t>(r) * slot_floats, x + row * ldx, row_bytes, &full[r]);
      }
    }
  float amax = 0.f;
  int slot = 0, par = 0;
  uint32_t phase = 0;
  for (index_t row = blockIdx.x; row < m; row += gridDim.x, par ^= 1) {
    tc::mbar_wait(&full[slot], phase, 20);
    const float* xs = slots + static_cast<size_t>(slot) * slot_floats;
    const uint32_t xs_s = tc::smem_u32(xs);
    if (xmax) {  // four independent maxima (a single chain exposes every load's latency)
      float am[4] = {0.f, 0.f, 0.f, 0.f};
      const int nv = n / 4;
      int q = threadIdx.x;
      for (; q + 3 * static_cast<int>(blockDim.x) < nv; q += 4 * blockDim.x) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w)
                       : "r"(xs_s + 16u * (q + k * blockDim.x)));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          am[k] = fmaxf(am[k], fmaxf(fmaxf(fabsf(v[k].x), fabsf(v[k].y)), fmaxf(fabsf(v[k].z), fabsf(v[k].w))));
      }
      for (; q < nv; q += blockDim.x) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(xs_s + 16u * q));
        am[0] = fmaxf(am[0], fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
      amax = fmaxf(amax, fmaxf(fmaxf(am[0], am[1]), fmaxf(am[2], am[3])));
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int g = 0; g < SMAX / 16; ++g) {
      if (16 * g < steps) {  // warp-uniform: the schedule's length
        float v[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const std::uint32_t w = e[8 * g + i];
          asm volatile("ld.shared.f32 %0, [%2];\n ld.shared.f32 %1, [%3];"
                       : "=f"(v[2 * i]), "=f"(v[2 * i + 1])
                       : "r"(xs_s + ((w & 0x7fffu) << 2)), "r"(xs_s + (((w >> 16) & 0x7fffu) << 2)));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const std::uint32_t w = e[8 * g + i];
          // the entry's sign flips the value's sign bit
          acc[(2 * i) & 3] += __uint_as_float(__float_as_uint(v[2 * i]) ^ ((w << 16) & 0x80000000u));
          acc[(2 * i + 1) & 3] += __uint_as_float(__float_as_uint(v[2 * i + 1]) ^ (w & 0x80000000u));
        }
      }
    }
    const float sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    if (P == 2 && part == 1) red[par * wps * 32 + col] = sum;
    __syncthreads();  // every warp is done with this slot (and the halves' sums are staged)
    if (threadIdx.x == 0) {
      const index_t next = row + static_cast<index_t>(ring) * gridDim.x;
      if (next < m) {
        tc::mbar_expect_tx(&full[slot], row_bytes);
        bulk_load(slots + static_cast<size_t>(slot) * slot_floats, x + next * ldx, row_bytes, &full[slot]);
      }
    }
    if (part == 0 && col < ldu)
      u[row * ldu + col] = col < l ? (P == 2 ? sum + red[par * wps * 32 + col] : sum) : 0.f;
    if (++slot == ring) {
      slot = 0;
      phase ^= 1u;
    }
  }
  if (xmax) {
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) atomicMax(xmax, __float_as_uint(amax));
  }
}

}  // namespace

index_t sparse_sketch_chunks(index_t n, int dtype) {
  const int kc = dtype == 4 ? chunk_cols<float>() : chunk_cols<double>();
  return (n + kc - 1) / kc;
}

void launch_omega_chunk_lists(cudaStream_t s, const double* omega, index_t n, index_t l, int dtype, int* counts,
                              int* ptr, std::uint32_t* ent) {
  const int kc = dtype == 4 ? chunk_cols<float>() : chunk_cols<double>();
  const int nchunks = static_cast<int>((n + kc - 1) / kc);
  const index_t cells = static_cast<index_t>(nchunks) * l;
  const unsigned g = static_cast<unsigned>((cells + 255) / 256);
  omega_chunk_count_kernel<<<g, 256, 0, s>>>(omega, n, l, kc, nchunks, counts);
  scan_kernel<<<1, 1024, 0, s>>>(counts, cells, ptr);
  const int neg_off = kRows * (dtype == 4 ? rows_per_lane<float>() : rows_per_lane<double>()) * (kc + 1);  // -X tile
  omega_chunk_fill_kernel<<<g, 256, 0, s>>>(omega, n, l, kc, nchunks, ptr, ent, neg_off, dtype);
}

template <typename T, int RPL, int MC>
void launch_sparse_sketch_v(cudaStream_t s, const T* x, index_t m, index_t n, index_t ldx, const int* ptr,
                            const std::uint32_t* ent, index_t l, T* u, index_t ldu, std::uint32_t* xmax, int num_sms) {
  constexpr int kc = chunk_cols<T>();
  constexpr int rows = kRows * RPL;
  const int nchunks = static_cast<int>((n + kc - 1) / kc);
  const size_t smem = sizeof(T) * ((2 * rows * (kc + 1) + 1) & ~1) + sizeof(int) * ((kWarps * MC + 1 + 3) & ~3) +
                      sizeof(std::uint32_t) * kEntCap;
  auto* kern = sparse_sketch_kernel<T, RPL, MC>;
  LPCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const index_t tiles = (m + rows - 1) / rows;
  const unsigned grid = static_cast<unsigned>(tiles < num_sms ? tiles : num_sms);
  kern<<<grid, kThreadsSO, smem, s>>>(x, m, n, ldx, ptr, ent, static_cast<int>(l), nchunks, u, ldu, xmax);
}

template <typename T>
void launch_sparse_sketch(cudaStream_t s, const T* x, index_t m, index_t n, index_t ldx, const int* ptr,
                          const std::uint32_t* ent, index_t l, T* u, index_t ldu, std::uint32_t* xmax, int num_sms) {
  if (m <= 0) return;
  if (ldu > 512 || ldu < l) throw Error(kInternal, "sparse sketch: l > 512");
  // up to 20 columns per warp (l <= 320): fp32 takes two rows per lane
  constexpr int RPL = rows_per_lane<T>();
  if (l <= kWarps * 20)
    launch_sparse_sketch_v<T, RPL, 20>(s, x, m, n, ldx, ptr, ent, l, u, ldu, xmax, num_sms);
  else
    launch_sparse_sketch_v<T, RPL, 32>(s, x, m, n, ldx, ptr, ent, l, u, ldu, xmax, num_sms);
}

void launch_u_planes_f16(cudaStream_t s, const float* u, index_t m, index_t ld, index_t npad, __half* hi, __half* lo,
                         index_t ldt, float* uinv) {
  if (m <= 0) return;
  const dim3 grid(static_cast<unsigned>((m + kUScaleRows - 1) / kUScaleRows), static_cast<unsigned>((npad + 31) / 32));
  u_planes_f16_kernel<<<grid, static_cast<unsigned>(kUScaleRows), 0, s>>>(u, m, ld, npad, hi, lo, ldt, uinv);
}

// ---- row gather: host schedule and launch -----------------------------------------

namespace {
constexpr int kRowSmemBudget = 200 * 1024;
int row_slot_floats(index_t n) { return static_cast<int>(((n + 31) / 32) * 32 + 32); }
}  // namespace

int row_gather_ring(index_t n) {
  const long long slot = 4LL * row_slot_floats(n);
  const long long r = (kRowSmemBudget - 64 - 4096) / slot;  // (mbarriers, the halves' sums)
  return static_cast<int>(r > 4 ? 4 : r);
}

bool row_gather_feasible(index_t m, index_t n, index_t ldx, index_t l) {
  return m > 0 && n % 4 == 0 && ldx % 4 == 0 && l <= 512 && row_slot_floats(n) <= 32768 && row_gather_ring(n) >= 2;
}


void launch_omega_col_lists(cudaStream_t s, const double* omega, index_t n, index_t l, int cap, int* cnt,
                            std::uint32_t* cols) {
  const unsigned blocks = static_cast<unsigned>((l + 7) / 8);
  omega_col_lists_kernel<<<blocks, 256, 0, s>>>(omega, n, l, cap, cnt, cols);
}

// One warp's bipartite multigraph (its 32 lanes = Omega columns x the 32 banks,
// an edge per nonzero: lane c -> bank j % 32) edge-coloured with Delta = the
// maximum degree colours (Koenig: bipartite multigraphs need no more), each
// colour a step in which the lanes read 32 distinct banks; an edge whose two
// ends have different first free colours a, b flips the a/b alternating path
// from its bank end first. out[s * 32 + lane]: the 16-bit entry of step s.
// Returns Delta, or -1 when it exceeds smax.
int schedule_warp(const std::vector<std::vector<std::uint32_t>>& lanes, int zbase, int smax, std::uint16_t* out) {
  int degl[32] = {}, degr[32] = {};
  std::vector<std::pair<int, std::uint32_t>> edges;  // (lane, entry)
  for (int c = 0; c < 32; ++c)
    for (std::uint32_t v : lanes[c]) {
      edges.emplace_back(c, v);
      ++degl[c];
      ++degr[(v & 0x7fffffffu) & 31u];
    }
  int delta = 0;
  for (int i = 0; i < 32; ++i) delta = std::max(delta, std::max(degl[i], degr[i]));
  if (delta > smax) return -1;
  const int E = static_cast<int>(edges.size());
  std::vector<int> at_l(32 * static_cast<size_t>(std::max(delta, 1)), -1), at_r(at_l.size(), -1), colour(E, -1);
  auto L = [&](int e) { return edges[e].first; };
  auto R = [&](int e) { return static_cast<int>((edges[e].second & 0x7fffffffu) & 31u); };
  std::vector<int> path;
  for (int e = 0; e < E; ++e) {
    const int u = L(e), v = R(e);
    int a = 0, b = 0;
    while (at_l[u * delta + a] >= 0) ++a;
    while (at_r[v * delta + b] >= 0) ++b;
    if (at_r[v * delta + a] >= 0) {
      // the a/b path from v: colour a at bank nodes, colour b at lane nodes
      path.clear();
      int node = v;
      bool bank_side = true;
      for (;;) {
        const int f = bank_side ? at_r[node * delta + a] : at_l[node * delta + b];
        if (f < 0) break;
        path.push_back(f);
        node = bank_side ? L(f) : R(f);
        bank_side = !bank_side;
      }
      for (int f : path) {
        at_l[L(f) * delta + colour[f]] = -1;
        at_r[R(f) * delta + colour[f]] = -1;
      }
      for (int f : path) {
        colour[f] = colour[f] == a ? b : a;
        at_l[L(f) * delta + colour[f]] = f;
        at_r[R(f) * delta + colour[f]] = f;
      }
    }
    colour[e] = a;
    at_l[u * delta + a] = e;
    at_r[v * delta + a] = e;
  }
  for (int st = 0; st < smax; ++st) {
    int freeb[32], nf = 0;
    for (int b = 0; b < 32; ++b)
      if (st >= delta || at_r[b * delta + st] < 0) freeb[nf++] = b;
    int k = 0;
    for (int c = 0; c < 32; ++c) {
      const int f = st < delta ? at_l[c * delta + st] : -1;
      std::uint32_t code;
      if (f >= 0) {
        const std::uint32_t v = edges[f].second;
        code = (v & 0x7fffu) | ((v >> 31) << 15);
      } else {
        code = static_cast<std::uint32_t>(zbase + freeb[k++]);  // a zero word in a bank nobody reads now
      }
      out[static_cast<size_t>(st) * 32 + c] = static_cast<std::uint16_t>(code);
    }
  }
  return delta;
}

int build_row_schedule(const int* cnt, const std::uint32_t* cols, int cap, index_t n, index_t l,
                       std::vector<std::uint32_t>& packed, int* smax_out, int* splits_out) {
  const int wps = static_cast<int>((l + 31) / 32);
  const int zbase = row_slot_floats(n) - 32;
  int need = 0;
  for (index_t c = 0; c < l; ++c) {
    if (cnt[c] > cap) return -1;
    need = std::max(need, cnt[c]);
  }
  // most warps first (the loads' latency), then the shortest unroll that fits
  // the schedule (bank degrees can exceed the column degrees)
  const int cand[][2] = {{64, 2}, {96, 2}, {64, 1}, {128, 1}, {192, 1}};
  for (const auto& cd : cand) {
    const int smax = cd[0], P = cd[1];
    if (wps * P * 32 > rows_max_threads(smax, P) || (P == 1 && need > smax)) continue;
    const index_t half = ((n + 1) / 2 + 31) / 32 * 32;  // j < half: first part
    const int warps = wps * P;
    std::vector<std::uint16_t> steps(static_cast<size_t>(warps) * smax * 32);
    int worst = 0;
    bool ok = true;
    for (int w = 0; w < warps && ok; ++w) {
      const int part = w / wps, g = w % wps;
      std::vector<std::vector<std::uint32_t>> lanes(32);
      for (int c = 0; c < 32; ++c) {
        const index_t col = static_cast<index_t>(g) * 32 + c;
        if (col >= l) continue;
        for (int i = 0; i < cnt[col]; ++i) {
          const std::uint32_t v = cols[col * cap + i];
          const index_t j = v & 0x7fffffffu;
          if (P == 1 || (part == 0) == (j < half)) lanes[c].push_back(v);
        }
      }
      const int d = schedule_warp(lanes, zbase, smax, steps.data() + static_cast<size_t>(w) * smax * 32);
      if (d < 0) ok = false;
      worst = std::max(worst, d);
    }
    if (!ok) continue;
    packed.assign(static_cast<size_t>(warps) * (smax / 2) * 32, 0u);
    for (int w = 0; w < warps; ++w)
      for (int i = 0; i < smax / 2; ++i)
        for (int c = 0; c < 32; ++c) {
          const std::uint16_t* base = steps.data() + static_cast<size_t>(w) * smax * 32;
          packed[(static_cast<size_t>(w) * (smax / 2) + i) * 32 + c] =
              static_cast<std::uint32_t>(base[(2 * i) * 32 + c]) |
              (static_cast<std::uint32_t>(base[(2 * i + 1) * 32 + c]) << 16);
        }
    *smax_out = smax;
    *splits_out = P;
    return worst;
  }
  return -1;
}

void launch_sparse_sketch_rows(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx,
                               const std::uint32_t* sched, int steps, int smax, int splits, index_t l, float* u,
                               index_t ldu, std::uint32_t* xmax, int num_sms) {
  if (m <= 0) return;
  if (ldu > ((l + 31) / 32) * 32) throw Error(kInternal, "row gather: ldu beyond the column warps");
  const int slot = row_slot_floats(n), ring = row_gather_ring(n);
  const int wps = static_cast<int>((l + 31) / 32);
  const size_t smem = static_cast<size_t>(ring) * slot * 4 + 64 + 2 * 4 * 32 * static_cast<size_t>(wps);
  const unsigned threads = static_cast<unsigned>(wps * 32 * splits);
  const unsigned grid = static_cast<unsigned>(m < num_sms ? m : num_sms);
  auto go = [&](auto kern) {
    LPCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, threads, smem, s>>>(x, m, static_cast<int>(n), ldx, sched, steps, slot, ring, static_cast<int>(l), u,
                                      ldu, xmax);
  };
  if (splits == 2 && smax == 64) go(sparse_sketch_rows_kernel<64, 2>);
  else if (splits == 2) go(sparse_sketch_rows_kernel<96, 2>);
  else if (smax == 64) go(sparse_sketch_rows_kernel<64, 1>);
  else if (smax == 128) go(sparse_sketch_rows_kernel<128, 1>);
  else go(sparse_sketch_rows_kernel<192, 1>);
}

template void launch_sparse_sketch<float>(cudaStream_t, const float*, index_t, index_t, index_t, const int*,
                                          const std::uint32_t*, index_t, float*, index_t, std::uint32_t*, int);
template void launch_sparse_sketch<double>(cudaStream_t, const double*, index_t, index_t, index_t, const int*,
                                           const std::uint32_t*, index_t, double*, index_t, std::uint32_t*, int);

}  // namespace lpca
