// tcgen05 split-TF32 GEMMs for fp32 data (sm_100a).
//
// Both X-passes of Lazy SPCA are tall-skinny products that stream X (m x n,
// fp32, row-major) once from HBM:
//   xw  : OUT = X W      (sketch U = X Omega, power U = X Z, transform Y = X V)
//   utx : F_part = U^T X (F formation and the power step's Z^T = U^T X)
// fp32-faithful results need more than one TF32 product (1xTF32
// misses the 1e-4 singular-value target), so every product is the 3-term split
//   a*b ~= a_hi*b_hi + a_lo*b_hi + a_hi*b_lo,  a_hi = tf32(a), a_lo = tf32(a - a_hi)
// accumulated in fp32 in TMEM. The small operand (W, or U^T) arrives pre-split
// as hi/lo planes; X is split in shared memory by four converter warps after
// TMA lands each stage, so X is read from HBM exactly once per pass.
//
// All UMMA operands are K-major with the 128 B swizzle (kind::tf32 with an
// MN-major operand produced no result on this part in our probes). For utx the
// reduction runs over X's rows, so the converter warps transpose each raw X
// tile into the K-major layout while splitting it; the swizzle makes those
// transposing stores bank-conflict free.
//
// Warp roles (one CTA per SM):
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer (one lane) + TMEM allocator
//   warps 2-5   split converters (128 threads)
//   warps 6-9   epilogue (TMEM -> registers -> global), one TMEM lane quarter each
// Pipelines: smem full/conv/empty ring (TMA -> convert -> MMA), and a
// double-buffered TMEM accumulator (MMA -> epilogue) so one tile's epilogue
// overlaps the next tile's MMAs.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <string>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace lpca {

namespace {

using namespace tc;

constexpr int kThreads = 320;
constexpr int kBM = 128;         // UMMA M
constexpr int kBK = 32;          // K per stage: 32 fp32 = one 128 B swizzle row
constexpr uint32_t kSmemBudget = 200 * 1024;
// The tensor core's fp32 accumulation rounds toward zero: measured bias about
// -5e-8 of the running sum per K=8 step (-2.6e-5 at K = 4096). MMAs therefore
// accumulate runs of at most kRunStages stages (K = 128, 16 steps) into a TMEM
// run buffer; epilogue warps fold runs into a TMEM-resident long accumulator
// with round-to-nearest fp32 adds, so the bias stays ~1e-6 for any K.
constexpr int kRunStages = 4;

__device__ __forceinline__ void split4(float4& v, float4& lo) {
  float4 h;
  h.x = tf32_trunc(v.x);
  h.y = tf32_trunc(v.y);
  h.z = tf32_trunc(v.z);
  h.w = tf32_trunc(v.w);
  lo.x = tf32_trunc(v.x - h.x);
  lo.y = tf32_trunc(v.y - h.y);
  lo.z = tf32_trunc(v.z - h.z);
  lo.w = tf32_trunc(v.w - h.w);
  v = h;
}

__device__ __forceinline__ void ring_advance(int& stage, uint32_t& phase, int S) {
  if (++stage == S) {
    stage = 0;
    phase ^= 1;
  }
}

// ------------------------------------------------------------------------------------
// xw: OUT[m x npad] = X[m x K] * W, W given as K-major hi/lo planes [npad][K].
// Persistent over 128-row tiles of X.
struct XwArgs {
  int m, kdim, npad, stages;
  int nrb;         // TMEM run buffers (2 when 3 * npad columns fit, else 1)
  uint32_t tmem_cols;
  int wstore;      // columns of `out` stored (<= npad)
  float* out;      // plain fp32, row-major, ld ldo (nullable)
  int ldo;
  float* out_hi;   // tf32 planes of OUT^T: [npad][ldh] (nullable)
  float* out_lo;
  int ldh;
};

__global__ void __launch_bounds__(kThreads, 1)
    xw_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmwh,
                 const __grid_constant__ CUtensorMap tmwl, XwArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages;
  constexpr uint32_t a_bytes = kBM * kBK * 4;  // 16 KB
  const uint32_t b_bytes = static_cast<uint32_t>(a.npad) * kBK * 4;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* full = bars;
  uint64_t* conv = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_tiles = (a.m + kBM - 1) / kBM;
  const int kiters = (a.kdim + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
    tma_prefetch(&tmx);
    tma_prefetch(&tmwh);
    tma_prefetch(&tmwl);
  }
  if (warp == 1) tmem_alloc(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < kiters; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1, 1);
          uint8_t* st = smem + stage * stage_bytes;
          mbar_expect_tx(&full[stage], a_bytes + 2 * b_bytes);
          tma_load_2d(st, &tmx, &full[stage], kb * kBK, tile * kBM);
          tma_load_2d(st + 2 * a_bytes, &tmwh, &full[stage], kb * kBK, 0);
          tma_load_2d(st + 2 * a_bytes + b_bytes, &tmwl, &full[stage], kb * kBK, 0);
          ring_advance(stage, phase, S);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(kBM, a.npad, 0, 0);
      int stage = 0, rc = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int kb0 = 0; kb0 < kiters; kb0 += kRunStages, ++rc) {
          const int b = rc % a.nrb;
          mbar_wait(&tempty[b], ((rc / a.nrb) & 1) ^ 1, 2);
          tc_fence_after();
          const uint32_t d = tmem_base + static_cast<uint32_t>(b * a.npad);
          const int kb1 = min(kiters, kb0 + kRunStages);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&conv[stage], phase, 3);
            tc_fence_after();
            const uint32_t ah = smem_u32(smem + stage * stage_bytes);
            const uint32_t al = ah + a_bytes, bh = ah + 2 * a_bytes, bl = bh + b_bytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
              const uint32_t off = kk * 32;  // 8 tf32 of K inside the 128 B swizzled row
              const uint64_t dah = sw128_desc(ah + off, 16, 1024), dal = sw128_desc(al + off, 16, 1024);
              const uint64_t dbh = sw128_desc(bh + off, 16, 1024), dbl = sw128_desc(bl + off, 16, 1024);
              mma_tf32(d, dah, dbh, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
              mma_tf32(d, dal, dbh, idesc, 1u);
              mma_tf32(d, dah, dbl, idesc, 1u);
            }
            mma_commit(&empty[stage]);
            ring_advance(stage, phase, S);
          }
          mma_commit(&tfull[b]);
        }
      }
    }
  } else if (warp < 6) {
    const int t = threadIdx.x - 64;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      for (int kb = 0; kb < kiters; ++kb) {
        mbar_wait(&full[stage], phase, 4);
        float4* hi = reinterpret_cast<float4*>(smem + stage * stage_bytes);
        float4* lo = reinterpret_cast<float4*>(smem + stage * stage_bytes + a_bytes);
#pragma unroll
        for (int i = 0; i < static_cast<int>(a_bytes / 16 / 128); ++i) {
          const int idx = t + 128 * i;
          float4 v = hi[idx], l4;
          split4(v, l4);
          hi[idx] = v;
          lo[idx] = l4;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[stage]);
        ring_advance(stage, phase, S);
      }
    }
  } else {
    const int q = warp & 3;
    const int runs = (kiters + kRunStages - 1) / kRunStages;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t lacc = lane_base + static_cast<uint32_t>(a.nrb * a.npad);  // long accumulator
    int rc = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int row = tile * kBM + q * 32 + lane;
      for (int r = 0; r < runs; ++r, ++rc) {
        const int b = rc % a.nrb;
        mbar_wait(&tfull[b], (rc / a.nrb) & 1, 5);
        tc_fence_after();
        const uint32_t racc = lane_base + static_cast<uint32_t>(b * a.npad);
        const bool first = r == 0, last = r == runs - 1;
        for (int c0 = 0; c0 < a.npad; c0 += 16) {
          float v[16];
          tmem_ld16(racc + c0, v);
          if (!first) {  // fold the run into the long accumulator, round-to-nearest
            float s[16];
            tmem_ld16(lacc + c0, s);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], s[i]);
          }
          if (!last) {
            tmem_st16(lacc + c0, v);
            continue;
          }
          if (row < a.m) {
            if (a.out_hi) {
              // transposed tf32 planes (OUT^T, [npad][ldh]): one row per lane, so
              // each column store of the warp is 32 consecutive floats (coalesced)
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float h = tf32_trunc(v[i]);
                a.out_hi[static_cast<size_t>(c0 + i) * a.ldh + row] = h;
                a.out_lo[static_cast<size_t>(c0 + i) * a.ldh + row] = tf32_trunc(v[i] - h);
              }
            }
            if (a.out) {
              float* po = a.out + static_cast<size_t>(row) * a.ldo;
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (c0 + i < a.wstore) po[c0 + i] = v[i];
            }
          }
        }
        if (!last) tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// ------------------------------------------------------------------------------------
// utx: part[s][j*l + r] = sum over the rows of split s of U[i, r] X[i, j].
// A = U^T from K-major tf32 planes [lpad][ldt] (as the sketch epilogue writes
// them), B = X^T tiles made K-major by the converters, K = rows of X. A CTA
// owns (n tile, row split); it accumulates `flush_rows` rows at a time in fp32
// in TMEM and folds each segment into its own fp64 slot of `part` (the first
// segment stores), so fp32 run lengths stay bounded and every cross-segment and
// cross-split sum is fp64 in a fixed order.
struct UtxArgs {
  int m, l, n;
  int mhalves;  // 1: l <= 128; 2: l <= 256 (two M = 128 halves sharing B)
  int bn;       // UMMA N = n tile (128 or 64)
  int rows_per_split, flush_rows, stages;
  uint32_t tmem_cols;
  double* part;
};

__global__ void __launch_bounds__(kThreads, 1)
    utx_tc_kernel(const __grid_constant__ CUtensorMap tmuh, const __grid_constant__ CUtensorMap tmul,
                  const __grid_constant__ CUtensorMap tmx, UtxArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages;
  const uint32_t a_half = kBM * kBK * 4;                      // 16 KB per M half
  const uint32_t a_bytes = a.mhalves * a_half;                // per plane
  const uint32_t b_bytes = static_cast<uint32_t>(a.bn) * kBK * 4;  // per plane, K-major
  const uint32_t raw_bytes = b_bytes;                         // raw X tile [32][bn]
  const uint32_t stage_bytes = 2 * a_bytes + 3 * b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* full = bars;
  uint64_t* conv = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = blockIdx.x * a.bn;
  const int split = blockIdx.y;
  const int r_begin = split * a.rows_per_split;
  const int r_end = min(a.m, r_begin + a.rows_per_split);
  const int nseg = r_end > r_begin ? (r_end - r_begin + a.flush_rows - 1) / a.flush_rows : 0;
  const uint32_t buf_cols = static_cast<uint32_t>(a.mhalves * a.bn);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
    tma_prefetch(&tmuh);
    tma_prefetch(&tmul);
    tma_prefetch(&tmx);
  }
  if (warp == 1) tmem_alloc(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int sg = 0; sg < nseg; ++sg) {
        const int s0 = r_begin + sg * a.flush_rows;
        const int s1 = min(r_end, s0 + a.flush_rows);
        for (int row = s0; row < s1; row += kBK) {
          mbar_wait(&empty[stage], phase ^ 1, 11);
          uint8_t* st = smem + stage * stage_bytes;
          mbar_expect_tx(&full[stage], 2 * a_bytes + raw_bytes);
          for (int h = 0; h < a.mhalves; ++h) {
            tma_load_2d(st + h * a_half, &tmuh, &full[stage], row, h * kBM);
            tma_load_2d(st + a_bytes + h * a_half, &tmul, &full[stage], row, h * kBM);
          }
          tma_load_2d(st + 2 * a_bytes + 2 * b_bytes, &tmx, &full[stage], n0, row);
          ring_advance(stage, phase, S);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(kBM, a.bn, 0, 0);
      int stage = 0, rc = 0;
      uint32_t phase = 0;
      for (int sg = 0; sg < nseg; ++sg) {
        const int s0 = r_begin + sg * a.flush_rows;
        const int s1 = min(r_end, s0 + a.flush_rows);
        for (int q0 = s0; q0 < s1; q0 += kRunStages * kBK, ++rc) {
          const int b = rc & 1;
          mbar_wait(&tempty[b], ((rc >> 1) & 1) ^ 1, 12);
          tc_fence_after();
          const int q1 = min(s1, q0 + kRunStages * kBK);
          for (int row = q0; row < q1; row += kBK) {
            mbar_wait(&conv[stage], phase, 13);
            tc_fence_after();
            const uint32_t ah = smem_u32(smem + stage * stage_bytes);
            const uint32_t al = ah + a_bytes, bh = ah + 2 * a_bytes, bl = bh + b_bytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
              const uint32_t off = kk * 32;
              const uint64_t dbh = sw128_desc(bh + off, 16, 1024), dbl = sw128_desc(bl + off, 16, 1024);
              for (int h = 0; h < a.mhalves; ++h) {
                const uint64_t dah = sw128_desc(ah + h * a_half + off, 16, 1024);
                const uint64_t dal = sw128_desc(al + h * a_half + off, 16, 1024);
                const uint32_t d = tmem_base + b * buf_cols + h * a.bn;
                mma_tf32(d, dah, dbh, idesc, (row != q0 || kk != 0) ? 1u : 0u);
                mma_tf32(d, dal, dbh, idesc, 1u);
                mma_tf32(d, dah, dbl, idesc, 1u);
              }
            }
            mma_commit(&empty[stage]);
            ring_advance(stage, phase, S);
          }
          mma_commit(&tfull[b]);
        }
      }
    }
  } else if (warp < 6) {
    // transpose + split: raw[k][j] (k = row in the stage, j = column of the n
    // tile) -> K-major SW128 planes, row j holding its 32 k values in 128 B with
    // 16 B chunk c stored at chunk (c ^ (j & 7)).
    const int t = threadIdx.x - 64;
    const int groups = 128 / a.bn;  // threads per n column (1 or 2)
    const int j = t % a.bn, g = t / a.bn;
    const int kper = kBK / groups;
    int stage = 0;
    uint32_t phase = 0;
    for (int sg = 0; sg < nseg; ++sg) {
      const int s0 = r_begin + sg * a.flush_rows;
      const int s1 = min(r_end, s0 + a.flush_rows);
      for (int row = s0; row < s1; row += kBK) {
        mbar_wait(&full[stage], phase, 14);
        uint8_t* st = smem + stage * stage_bytes;
        const float* raw = reinterpret_cast<const float*>(st + 2 * a_bytes + 2 * b_bytes);
        uint8_t* bh = st + 2 * a_bytes;
        uint8_t* bl = bh + b_bytes;
        for (int c4 = 0; c4 < kper / 4; ++c4) {
          const int k0 = g * kper + c4 * 4;
          float4 v = make_float4(raw[(k0 + 0) * a.bn + j], raw[(k0 + 1) * a.bn + j],
                                 raw[(k0 + 2) * a.bn + j], raw[(k0 + 3) * a.bn + j]);
          float4 l4;
          split4(v, l4);
          const uint32_t off = static_cast<uint32_t>(j) * 128 + ((((k0 >> 2) ^ (j & 7))) << 4);
          *reinterpret_cast<float4*>(bh + off) = v;
          *reinterpret_cast<float4*>(bl + off) = l4;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[stage]);
        ring_advance(stage, phase, S);
      }
    }
  } else {
    const int q = warp & 3;
    double* dst = a.part + static_cast<size_t>(split) * a.l * a.n;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t lacc = lane_base + 2 * buf_cols;  // long accumulator
    int rc = 0;
    for (int sg = 0; sg < nseg; ++sg) {
      const int s0 = r_begin + sg * a.flush_rows;
      const int s1 = min(r_end, s0 + a.flush_rows);
      const int runs = (s1 - s0 + kRunStages * kBK - 1) / (kRunStages * kBK);
      for (int rr = 0; rr < runs; ++rr, ++rc) {
        const int b = rc & 1;
        mbar_wait(&tfull[b], (rc >> 1) & 1, 15);
        tc_fence_after();
        const bool first = rr == 0, last = rr == runs - 1;
        for (int h = 0; h < a.mhalves; ++h) {
          const int r = h * kBM + q * 32 + lane;
          const uint32_t racc = lane_base + b * buf_cols + h * a.bn;
          const uint32_t lh = lacc + h * a.bn;
          for (int c0 = 0; c0 < a.bn; c0 += 16) {
            float v[16];
            tmem_ld16(racc + c0, v);
            if (!first) {
              float s[16];
              tmem_ld16(lh + c0, s);
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], s[i]);
            }
            if (!last) {
              tmem_st16(lh + c0, v);
              continue;
            }
            if (r < a.l) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const int jj = n0 + c0 + i;
                if (jj < a.n) {
                  double* p = dst + static_cast<size_t>(jj) * a.l + r;
                  *p = sg == 0 ? static_cast<double>(v[i]) : *p + static_cast<double>(v[i]);
                }
              }
            }
          }
        }
        if (!last) tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// ---- host side ----------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    LPCA_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw Error(kCuda, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp32 tensor map: `inner` contiguous elements per row, `outer` rows, row
// pitch `ld` elements, box {box_inner, box_outer}.
CUtensorMap map_2d(const float* base, index_t inner, index_t outer, index_t ld, uint32_t box_inner,
                   uint32_t box_outer, bool swizzle128) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

uint32_t tmem_cols_for(uint32_t need) {
  uint32_t c = 32;
  while (c < need) c <<= 1;
  return c;
}

int utx_bn(index_t l) { return l <= 128 ? 128 : 64; }

}  // namespace

bool tc_xw_supported(index_t n, index_t wpad) { return wpad >= 16 && wpad <= 256 && wpad % 16 == 0 && n >= 1; }

bool tc_utx_supported(index_t l, index_t n) { return l >= 1 && l <= 256 && n >= 1; }

void launch_xw_tc_planes(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx,
                         const float* w_hi, const float* w_lo, index_t wpad, index_t ldw, float* out,
                         index_t ldo, index_t wstore, float* out_hi, float* out_lo, index_t ldh,
                         int num_sms) {
  if (m <= 0) return;
  if (!tc_xw_supported(n, wpad)) throw Error(kInternal, "xw_tc: unsupported shape");
  if (ldx % 4 || ldw % 4 || (out_hi && ldh % 4))
    throw Error(kInternal, "xw_tc: leading dimensions must be multiples of 4 floats");
  const CUtensorMap tx = map_2d(x, n, m, ldx, 32, kBM, true);
  const CUtensorMap th = map_2d(w_hi, n, wpad, ldw, 32, static_cast<uint32_t>(wpad), true);
  const CUtensorMap tl = map_2d(w_lo, n, wpad, ldw, 32, static_cast<uint32_t>(wpad), true);
  XwArgs a{};
  a.m = static_cast<int>(m);
  a.kdim = static_cast<int>(n);
  a.npad = static_cast<int>(wpad);
  const uint32_t stage_bytes = 2 * kBM * kBK * 4 + 2 * static_cast<uint32_t>(wpad) * kBK * 4;
  a.stages = static_cast<int>(kSmemBudget / stage_bytes);
  if (a.stages > 6) a.stages = 6;
  a.nrb = 3 * wpad <= 512 ? 2 : 1;
  a.tmem_cols = tmem_cols_for(static_cast<uint32_t>((a.nrb + 1) * wpad));
  a.wstore = static_cast<int>(wstore);
  a.out = out;
  a.ldo = static_cast<int>(ldo);
  a.out_hi = out_hi;
  a.out_lo = out_lo;
  a.ldh = static_cast<int>(ldh);
  const size_t smem = static_cast<size_t>(a.stages) * stage_bytes + 1024 + 256;
  LPCA_CUDA(cudaFuncSetAttribute(xw_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const index_t tiles = ceil_div(m, kBM);
  const int grid = static_cast<int>(tiles < num_sms ? tiles : num_sms);
  xw_tc_kernel<<<grid, kThreads, smem, s>>>(tx, th, tl, a);
}

void launch_xw_tc(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx, const float* w_hi,
                  const float* w_lo, index_t wpad, index_t ldw, float* out, index_t ldo, int num_sms) {
  launch_xw_tc_planes(s, x, m, n, ldx, w_hi, w_lo, wpad, ldw, out, ldo, wpad, nullptr, nullptr, 0, num_sms);
}

index_t utx_tc_splits(index_t m, index_t l, index_t n, int num_sms, index_t* rows_per_split) {
  const index_t ntiles = ceil_div(n, utx_bn(l));
  index_t splits = num_sms / ntiles;
  if (splits < 1) splits = 1;
  const index_t max_splits = ceil_div(m, kBK);
  if (splits > max_splits) splits = max_splits;
  index_t rps = round_up(ceil_div(m, splits), kBK);
  splits = ceil_div(m, rps);
  *rows_per_split = rps;
  return splits;
}

void launch_utx_tc_planes(cudaStream_t s, const float* ut_hi, const float* ut_lo, index_t ldt, const float* x,
                          index_t ldx, index_t m, index_t l, index_t n, double* part, int num_sms) {
  if (!tc_utx_supported(l, n)) throw Error(kInternal, "utx_tc: unsupported shape");
  if (ldt % 4 || ldx % 4) throw Error(kInternal, "utx_tc: leading dimensions must be multiples of 4 floats");
  UtxArgs a{};
  a.m = static_cast<int>(m);
  a.l = static_cast<int>(l);
  a.n = static_cast<int>(n);
  a.mhalves = l <= 128 ? 1 : 2;
  a.bn = utx_bn(l);
  index_t rps = 0;
  const index_t splits = utx_tc_splits(m, l, n, num_sms, &rps);
  a.rows_per_split = static_cast<int>(rps);
  a.flush_rows = 8192;
  const uint32_t stage_bytes = 2 * static_cast<uint32_t>(a.mhalves) * kBM * kBK * 4 +
                               3 * static_cast<uint32_t>(a.bn) * kBK * 4;
  a.stages = static_cast<int>(kSmemBudget / stage_bytes);
  if (a.stages > 6) a.stages = 6;
  a.tmem_cols = tmem_cols_for(3 * static_cast<uint32_t>(a.mhalves * a.bn));
  a.part = part;
  const index_t lrows = round_up(l, 16);  // rows of the U^T planes
  const CUtensorMap th = map_2d(ut_hi, m, lrows, ldt, 32, kBM, true);
  const CUtensorMap tl = map_2d(ut_lo, m, lrows, ldt, 32, kBM, true);
  const CUtensorMap tx = map_2d(x, n, m, ldx, static_cast<uint32_t>(a.bn), kBK, false);
  const size_t smem = static_cast<size_t>(a.stages) * stage_bytes + 1024 + 256;
  LPCA_CUDA(cudaFuncSetAttribute(utx_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  dim3 grid(static_cast<unsigned>(ceil_div(n, a.bn)), static_cast<unsigned>(splits));
  utx_tc_kernel<<<grid, kThreads, smem, s>>>(th, tl, tx, a);
}

void launch_utx_tc(cudaStream_t, const float*, index_t, const float*, index_t, index_t, index_t, index_t,
                   index_t, double*, int) {
  throw Error(kInternal, "use launch_utx_tc_planes (U^T arrives as tf32 hi/lo planes)");
}

}  // namespace lpca
