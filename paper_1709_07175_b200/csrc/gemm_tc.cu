// tcgen05 split-TF32 GEMMs for fp32 data (sm_100a).
//
// Both X-passes of Lazy SPCA are tall-skinny products that stream X (m x n,
// fp32, row-major) once from HBM:
//   XW  : OUT = X W        (sketch U = X Omega, power U = X Z, transform Y = X V)
//   XTU : F^T = X^T U      (F formation and the power step's Z = X^T U)
// fp32-faithful results need more than one TF32 product (1xTF32
// misses the 1e-4 singular-value target), so every product is the 3-term split
//   a*b ~= a_hi*b_hi + a_lo*b_hi + a_hi*b_lo,  a_hi = tf32(a), a_lo = tf32(a - a_hi).
//
// Operand placement (one kernel template for both passes):
//   A = the X tile, M = 128 (XW: 128 rows of X; XTU: 128 columns of X), read
//       once from HBM by TMA, split into tf32 hi/lo by four converter warps and
//       written straight into a TMEM ring with tcgen05.st (the MMA reads A from
//       TMEM, the "TS" form) — XTU's converters transpose while they split.
//   B = the small operand's pre-split hi/lo planes, K-major [N][K] in shared
//       memory (XW: W^T planes; XTU: U^T planes), N = round_up(w, 16).
// With A in TMEM the tensor core reads only B from shared memory (42 KB per
// 32-deep stage at N = 112, plus the converters' 16 KB), under the MMA time of
// the stage; with A in shared memory as well it was smem-bandwidth bound
// (90 KB of operand reads per stage; ncu: tensor pipe 51% active).
//
// Accumulation: the tensor core's fp32 accumulation rounds toward zero
// (measured bias ~ -5e-8 of the running sum per K=8 step, -2.6e-5 at K=4096).
// MMAs accumulate runs of kRunStages stages (K = 128) into a TMEM run buffer;
// epilogue warps fold each run into a TMEM-resident long accumulator with
// round-to-nearest fp32 adds, so the bias stays ~1e-6 for any K.
//
// Warp roles (one CTA per SM, persistent over work items):
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer (one lane) + TMEM allocator
//   warps 2-5   split converters: smem X tile -> TMEM A hi/lo (one lane quarter each)
//   warps 6-9   epilogue: TMEM -> registers -> global (one lane quarter each)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace lpca {

namespace {

using namespace tc;

constexpr int kThreads = 320;
constexpr int kBM = 128;  // UMMA M (A rows = TMEM lanes)
constexpr int kBK = 32;   // K per stage
constexpr int kRunStages = 4;
constexpr uint32_t kSmemBudget = 200 * 1024;

enum Mode : int { kXW = 0, kXTU = 1 };

struct TcArgs {
  int m, n;          // X is m x n
  int npad;          // UMMA N
  int stages;        // smem ring depth
  int aslots;        // TMEM A ring depth (each slot: 64 columns, hi + lo)
  int nrb;           // TMEM run buffers
  uint32_t tmem_cols;
  int items;         // work items (XW: row tiles; XTU: n tiles x row chunks)
  int chunks;        // XTU: row chunks per n tile
  int chunk_rows;    // XTU: rows per chunk (multiple of kBK)
  // XW outputs
  int wstore;        // columns of `out` stored
  float* out;        // plain fp32 row-major, ld ldo (nullable)
  int ldo;
  float* out_hi;     // tf32 planes of OUT^T: [npad][ldh] (nullable)
  float* out_lo;
  int ldh;
  // XTU output: part[chunk][j * l + r] (fp64), r < l
  double* part;
  int l;
};

__device__ __forceinline__ void ring_advance(int& stage, uint32_t& phase, int S) {
  if (++stage == S) {
    stage = 0;
    phase ^= 1;
  }
}

// Work item -> (X tile origin along M, K range).
template <int kMode>
__device__ __forceinline__ void item_coords(const TcArgs& a, int item, int& t0, int& k0, int& k1) {
  if (kMode == kXW) {
    t0 = item * kBM;  // first row
    k0 = 0;
    k1 = a.n;
  } else {
    // chunk-major: the CTAs running together share row chunks, so the U^T
    // planes of those rows are re-read from L2 by every n tile, not from HBM
    const int ntiles = (a.n + kBM - 1) / kBM;
    const int nt = item % ntiles, ch = item / ntiles;
    t0 = nt * kBM;  // first column
    k0 = ch * a.chunk_rows;
    k1 = min(a.m, k0 + a.chunk_rows);
  }
}

template <int kMode>
__global__ void __launch_bounds__(kThreads, 1)
    tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmbh,
              const __grid_constant__ CUtensorMap tmbl, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the shared array (an integer round
  // trip would lose the address space and turn every access generic)
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  const int S = a.stages, AS = a.aslots;
  constexpr uint32_t x_bytes = kBM * kBK * 4;  // 16 KB X tile
  const uint32_t b_bytes = static_cast<uint32_t>(a.npad) * kBK * 4;
  const uint32_t stage_bytes = x_bytes + 2 * b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* full = bars;            // S: TMA landed (X + B planes)
  uint64_t* empty = full + S;       // S: MMAs done with the smem stage
  uint64_t* conv = empty + S;       // AS: A slot written to TMEM
  uint64_t* aempty = conv + AS;     // AS: MMAs done with the A slot
  uint64_t* tfull = aempty + AS;    // 2: run accumulated
  uint64_t* tempty = tfull + 2;     // 2: run buffer drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t a_col0 = static_cast<uint32_t>((a.nrb + 1) * a.npad);  // A ring after the accumulators

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(&conv[s], 4);
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
    tma_prefetch(&tmx);
    tma_prefetch(&tmbh);
    tma_prefetch(&tmbl);
  }
  if (warp == 1) tmem_alloc(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        int t0, k0, k1;
        item_coords<kMode>(a, item, t0, k0, k1);
        for (int k = k0; k < k1; k += kBK) {
          mbar_wait(&empty[stage], phase ^ 1, 1);
          uint8_t* st = smem + stage * stage_bytes;
          mbar_expect_tx(&full[stage], x_bytes + 2 * b_bytes);
          if (kMode == kXW)
            tma_load_2d(st, &tmx, &full[stage], k, t0);  // rows t0.., cols k..
          else
            tma_load_2d(st, &tmx, &full[stage], t0, k);  // cols t0.., rows k..
          tma_load_2d(st + x_bytes, &tmbh, &full[stage], k, 0);
          tma_load_2d(st + x_bytes + b_bytes, &tmbl, &full[stage], k, 0);
          ring_advance(stage, phase, S);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp walks the schedule (so every value below is warp-uniform)
    // and one elected lane issues each stage's 12 MMAs + commits in one go.
    const uint32_t idesc = idesc_tf32(kBM, a.npad, 0, 0);
    const uint64_t desc0 = sw128_desc(smem_u32(smem) + x_bytes, 16, 1024);
    int stage = 0, aslot = 0, rc = 0;
    uint32_t phase = 0, aphase = 0;
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
      int t0, k0, k1;
      item_coords<kMode>(a, item, t0, k0, k1);
      for (int q0 = k0; q0 < k1; q0 += kRunStages * kBK, ++rc) {
        const int b = rc % a.nrb;
        mbar_wait(&tempty[b], ((rc / a.nrb) & 1) ^ 1, 2);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(b * a.npad);
        const int q1 = min(k1, q0 + kRunStages * kBK);
        for (int k = q0; k < q1; k += kBK) {
          mbar_wait(&conv[aslot], aphase, 3);
          mbar_wait(&full[stage], phase, 3);
          tc_fence_after();
          // descriptor start address advances in 16 B units
          const uint64_t bh = desc0 + static_cast<uint64_t>((stage * stage_bytes) >> 4);
          const uint64_t bl = bh + static_cast<uint64_t>(b_bytes >> 4);
          const uint32_t at = tmem_base + a_col0 + static_cast<uint32_t>(aslot * 64);
          if (elect_one()) {
            mma_stage_ts(d, at, at + 32, bh, bl, idesc, k != q0 ? 1u : 0u);
            mma_commit(&empty[stage]);
            mma_commit(&aempty[aslot]);
          }
          __syncwarp();
          ring_advance(stage, phase, S);
          ring_advance(aslot, aphase, AS);
        }
        if (elect_one()) mma_commit(&tfull[b]);
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ---------------- converters: smem X -> TMEM A (hi, lo) ----------------
    const int q = warp & 3;
    const int i = q * 32 + lane;  // A row = TMEM lane
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    int stage = 0, aslot = 0;
    uint32_t phase = 0, aphase = 0;
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
      int t0, k0, k1;
      item_coords<kMode>(a, item, t0, k0, k1);
      for (int k = k0; k < k1; k += kBK) {
        mbar_wait(&full[stage], phase, 4);
        mbar_wait(&aempty[aslot], aphase ^ 1, 4);
        tc_fence_after();
        const uint8_t* xt = smem + stage * stage_bytes;
        float v[32];
        if (kMode == kXW) {
          // row i of a 128 B-swizzled [128][32] tile: 16 B chunk c at (c ^ (i & 7))
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 f = *reinterpret_cast<const float4*>(xt + i * 128 + ((c ^ (i & 7)) << 4));
            v[4 * c] = f.x;
            v[4 * c + 1] = f.y;
            v[4 * c + 2] = f.z;
            v[4 * c + 3] = f.w;
          }
        } else {
          // column i of a plain [32][128] tile
          const float* raw = reinterpret_cast<const float*>(xt);
#pragma unroll
          for (int kk = 0; kk < 32; ++kk) v[kk] = raw[kk * kBM + i];
        }
        float hi[32], lo[32];
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) {
          hi[kk] = tf32_trunc(v[kk]);
          lo[kk] = tf32_trunc(v[kk] - hi[kk]);
        }
        const uint32_t at = lane_base + a_col0 + static_cast<uint32_t>(aslot * 64);
        tmem_st32(at, hi);
        tmem_st32(at + 32, lo);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[aslot]);
        ring_advance(stage, phase, S);
        ring_advance(aslot, aphase, AS);
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t lacc = lane_base + static_cast<uint32_t>(a.nrb * a.npad);
    int rc = 0;
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
      int t0, k0, k1;
      item_coords<kMode>(a, item, t0, k0, k1);
      const int runs = (k1 - k0 + kRunStages * kBK - 1) / (kRunStages * kBK);
      const int row = t0 + q * 32 + lane;  // XW: X row; XTU: X column j
      for (int r = 0; r < runs; ++r, ++rc) {
        const int b = rc % a.nrb;
        mbar_wait(&tfull[b], (rc / a.nrb) & 1, 5);
        tc_fence_after();
        const uint32_t racc = lane_base + static_cast<uint32_t>(b * a.npad);
        const bool first = r == 0, last = r == runs - 1;
        for (int c0 = 0; c0 < a.npad; c0 += 16) {
          float v[16];
          tmem_ld16(racc + c0, v);
          if (!first) {
            float s[16];
            tmem_ld16(lacc + c0, s);
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = __fadd_rn(v[e], s[e]);
          }
          if (!last) {
            tmem_st16(lacc + c0, v);
            continue;
          }
          if (kMode == kXW) {
            if (row < a.m) {
              if (a.out_hi) {
                // transposed planes [npad][ldh]: one row per lane -> coalesced columns
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const float h = tf32_trunc(v[e]);
                  a.out_hi[static_cast<size_t>(c0 + e) * a.ldh + row] = h;
                  a.out_lo[static_cast<size_t>(c0 + e) * a.ldh + row] = tf32_trunc(v[e] - h);
                }
              }
              if (a.out) {
                float* po = a.out + static_cast<size_t>(row) * a.ldo;
#pragma unroll
                for (int e = 0; e < 16; ++e)
                  if (c0 + e < a.wstore) po[c0 + e] = v[e];
              }
            }
          } else if (row < a.n) {
            // F^T row j = F column j: part[chunk][j * l + r]
            double* p = a.part + static_cast<size_t>(item / ((a.n + kBM - 1) / kBM)) * a.l * a.n +
                        static_cast<size_t>(row) * a.l;
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (c0 + e < a.l) p[c0 + e] = static_cast<double>(v[e]);
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

#include "tc_pair.cuh"

// ---- host side ----------------------------------------------------------------------
// 2-SM pair kernels (tc_pair.cuh) unless LPCA_TC_PAIR=0.
bool pair_mode() {
  static const bool on = [] {
    const char* e = getenv("LPCA_TC_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

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

// 2-D tensor map of fp32 (esize 4) or fp16 (esize 2) elements: `inner`
// contiguous elements per row, `outer` rows, row pitch `ld` elements, box
// {box_inner, box_outer}.
CUtensorMap map_2d(const void* base, index_t inner, index_t outer, index_t ld, uint32_t box_inner,
                   uint32_t box_outer, bool swizzle128, int esize = 4) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(
      &m, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base),
      dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

uint32_t tmem_cols_for(uint32_t need) {
  uint32_t c = 32;
  while (c < need) c <<= 1;
  return c;
}

// TMEM plan: nrb run buffers + long accumulator + A ring (64 columns per slot).
bool plan_tmem(int npad, int& nrb, int& aslots, uint32_t& cols) {
  const int max_nrb = env_int("LPCA_TC_NRB", 2) > 2 ? 2 : env_int("LPCA_TC_NRB", 2);  // tfull/tempty hold 2
  const int max_as = env_int("LPCA_TC_ASLOTS", 2);
  for (int r = max_nrb; r >= 1; --r) {
    const int acc = (r + 1) * npad;
    const int slots = (512 - acc) / 64;
    if (slots >= 1) {
      nrb = r;
      aslots = slots > max_as ? max_as : slots;
      cols = tmem_cols_for(static_cast<uint32_t>(acc + 64 * aslots));
      return true;
    }
  }
  return false;
}
bool plan_tmem(int npad, TcArgs& a) { return plan_tmem(npad, a.nrb, a.aslots, a.tmem_cols); }

constexpr uint32_t kPairSmemBudget = 208 * 1024;

template <int kMode, bool kHalf>
void launch_pair(cudaStream_t s, const CUtensorMap& tx, const CUtensorMap& th, const CUtensorMap& tl, PairArgs& a,
                 int num_sms, cudaEvent_t ev_pre = nullptr, cudaEvent_t ev_post = nullptr) {
  if (!plan_tmem(a.npad, a.nrb, a.aslots, a.tmem_cols)) throw Error(kInternal, "tc pair: TMEM plan failed");
  // wide fp16 slices (one full A slot left): two half-stage slots in its place,
  // so conversion and MMA overlap (LPCA_TC_HALFSLOTS=0 keeps the single slot)
  // wide slices keep one full slot's worth of A columns: cut it into quarter
  // slots (K = 16), so a freed quarter is refilled while the MMAs read the other
  // three (LPCA_TC_SLOTDIV = 1 / 2 / 4 forces full / half / quarter slots)
  const int div = env_int("LPCA_TC_SLOTDIV", a.aslots == 1 ? 4 : 1);
  a.half_slots = kHalf && (div == 2 || div == 4) ? div : 0;
  if (a.half_slots == 4) {  // quarter slots fill every free TMEM column (up to 8 of them)
    const int acc = (a.nrb + 1) * a.npad;
    const int q = (512 - acc) / 16;
    a.aslots = q > 8 ? 8 : q;
    a.tmem_cols = tmem_cols_for(static_cast<uint32_t>(acc + 16 * a.aslots));
  } else if (a.half_slots) {
    a.aslots *= a.half_slots;
  }
  const uint32_t bk = kHalf ? 64 : 32;
  const uint32_t stage_bytes = kBM * bk * 4 + static_cast<uint32_t>(a.npad) * 128;  // X + half B (hi, lo)
  a.stages = static_cast<int>(kPairSmemBudget / stage_bytes);
  if (a.stages > 8) a.stages = 8;
  if (kHalf && kMode == kXW && a.scan == 1 && a.run_stages > a.stages) a.run_stages = a.stages;  // a scanned run fits the ring
  if (kHalf && kMode == kXTU && a.scan)  // a scanned run must fit the stage ring: runs of 2^k stages within a block
    while (a.run_stages > a.stages) a.run_stages /= 2;
  const size_t smem = static_cast<size_t>(a.stages) * stage_bytes + 1024 + 512 + (kMaxEpiWarps + 3) * 4 * a.npad +
                      kRscRing * 4 * kBM + 2 * 4 * kBM;  // red, gsc, xbuf, xrow
  LPCA_CUDA(cudaFuncSetAttribute(tc2_kernel<kMode, kHalf, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const int pairs = a.items < num_sms / 2 ? a.items : num_sms / 2;
  if constexpr (kMode == kXW) {
    // wide slices: 8 epilogue warps. LPCA_TC_CONV=8 (8 converters, fp16 with
    // quarter A slots) or 84 (8 converters, 4 epilogue warps): the MMA's wait
    // for converted A falls 39% -> 20% of its time, but at configs[2]'s
    // power-capped clocks the passes do not get faster, so 4
    // converters stay the default
    const int conv = kHalf && a.half_slots == 4 ? env_int("LPCA_TC_CONV", 4) : 4;
    auto go = [&](auto kern, int threads) {
      LPCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      if (ev_pre) LPCA_CUDA(cudaEventRecord(ev_pre, s));
      kern<<<2 * pairs, threads, smem, s>>>(tx, th, tl, a);
      if (ev_post) LPCA_CUDA(cudaEventRecord(ev_post, s));
    };
    if (a.npad > 168) {
      if constexpr (kHalf) {
        if (conv == 8) return go(tc2_kernel<kMode, kHalf, 8, 8>, pair_threads(8, 8));
        if (conv == 84) return go(tc2_kernel<kMode, kHalf, 4, 8>, pair_threads(8, 4));
      }
      return go(tc2_kernel<kMode, kHalf, 8, 4>, pair_threads(4, 8));
    }
  }
  if (ev_pre) LPCA_CUDA(cudaEventRecord(ev_pre, s));
  tc2_kernel<kMode, kHalf, 4><<<2 * pairs, pair_threads(4, 4), smem, s>>>(tx, th, tl, a);
  if (ev_post) LPCA_CUDA(cudaEventRecord(ev_post, s));
}

template <int kMode>
void launch(cudaStream_t s, const CUtensorMap& tx, const CUtensorMap& th, const CUtensorMap& tl, TcArgs& a,
            int grid) {
  const uint32_t stage_bytes = kBM * kBK * 4 + 2 * static_cast<uint32_t>(a.npad) * kBK * 4;
  a.stages = static_cast<int>(kSmemBudget / stage_bytes);
  if (a.stages > 6) a.stages = 6;
  const size_t smem = static_cast<size_t>(a.stages) * stage_bytes + 1024 + 256;
  LPCA_CUDA(cudaFuncSetAttribute(tc_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  tc_kernel<kMode><<<grid, kThreads, smem, s>>>(tx, th, tl, a);
}

}  // namespace

bool tc_xw_supported(index_t n, index_t wpad) {
  if (pair_mode()) return wpad >= 16 && wpad % 16 == 0 && n >= 1 && wpad <= 4096;  // sliced above pair_max_n()
  int nrb, as;
  uint32_t cols;
  return wpad >= 16 && wpad <= 256 && wpad % 16 == 0 && n >= 1 && plan_tmem(static_cast<int>(wpad), nrb, as, cols);
}

bool tc_utx_supported(index_t l, index_t n) { return l >= 1 && n >= 1 && tc_xw_supported(1, round_up(l, 16)); }

bool tc_pair_mode() { return pair_mode(); }

// Widths above this run as column slices over X (one launch per slice): TMEM
// holds two run buffers, the long accumulator and two A slots only for N <= 128.
int pair_max_n() { return env_int("LPCA_TC_MAXN", 128); }

// Column slices of a padded width: ceil(wpad / 224) slices of equal 16-multiples.
// Each slice is one more pass over X (and one more fp16 split of it), so fewer
// slices win now that the quarter A slots fill whatever TMEM a wide slice
// leaves: c4 (l = 300) X W as two 152-wide slices 74 ms against three 112-wide
// 88 ms (round 1, before quarter slots, 128-wide slices had won above 224).
// LPCA_TC_MAXN sets another maximum (A/B).
int slice_width(index_t wpad, bool) {
  int mx = 224;
  if (std::getenv("LPCA_TC_MAXN")) mx = pair_max_n();
  const index_t nsl = ceil_div(wpad, static_cast<index_t>(mx));
  return static_cast<int>(round_up(ceil_div(wpad, nsl), 16));
}

void launch_xw_pair(cudaStream_t s, const XwPairArgs& p, int num_sms) {
  if (p.m <= 0) return;
  if (p.wpad < 16 || p.wpad % 16 || p.n < 1) throw Error(kInternal, "xw_pair: unsupported shape");
  if (p.ldx % 4 || (p.half ? p.ldw % 8 : p.ldw % 4) || (p.out_hi && p.ldh % 4) || (p.uh && p.ldh % 8))
    throw Error(kInternal, "xw_pair: leading dimensions must be 16-byte multiples");
  if (p.half && !p.winv) throw Error(kInternal, "xw_pair: fp16 encoding needs the W scales");
  const int esz = p.half ? 2 : 4;
  const int sw = slice_width(p.wpad, false);
  for (index_t c0 = 0; c0 < p.wpad; c0 += sw) {
    const int wc = static_cast<int>(p.wpad - c0 < sw ? p.wpad - c0 : sw);
    PairArgs a{};
    a.m = static_cast<int>(p.m);
    a.n = static_cast<int>(p.n);
    a.npad = wc;
    a.items = static_cast<int>(ceil_div(p.m, 2 * kBM));
    // fp16 runs: K = 1024 (16 stages; the fold into the long accumulator
    // every 512 cost ~3% of a configs[2] step at the power cap, for 1.2-1.5x
    // smaller singular-value errors, all far inside the 1e-4 target); the
    // scanned sketch clamps to the stage ring. tf32: K = 256.
    a.run_stages = env_int("LPCA_TC_RUN", p.half ? 16 : 8);
    a.scan = p.half && !p.xmax_in && !(p.xmax_val > 0.0f) ? (p.ovf ? 2 : 1) : 0;
    a.ovf = p.ovf;
    a.wlo_nz = p.half ? p.wlo_nz : nullptr;
    a.xmax_in = p.xmax_in;
    a.xmax_val = p.xmax_val;
    a.xmax_out = c0 == 0 ? p.xmax_out : nullptr;
    a.winv = p.winv ? p.winv + c0 : nullptr;
    const index_t st = p.wstore - c0;
    a.wstore = static_cast<int>(st < 0 ? 0 : (st < wc ? st : wc));
    a.out = p.out ? p.out + c0 : nullptr;
    a.ldo = static_cast<int>(p.ldo);
    a.out_hi = p.out_hi ? p.out_hi + c0 * p.ldh : nullptr;
    a.out_lo = p.out_lo ? p.out_lo + c0 * p.ldh : nullptr;
    a.uh = p.uh ? p.uh + c0 * p.ldh : nullptr;
    a.ul = p.ul ? p.ul + c0 * p.ldh : nullptr;
    a.uinv = p.uinv ? p.uinv + c0 : nullptr;
    a.uinv_ld = static_cast<int>(p.wpad);
    a.ldh = static_cast<int>(p.ldh);
    const uint32_t brows = static_cast<uint32_t>(wc / 2);
    const char* wh = static_cast<const char*>(p.w_hi) + c0 * p.ldw * esz;
    const char* wl = static_cast<const char*>(p.w_lo) + c0 * p.ldw * esz;
    const CUtensorMap tx = map_2d(p.x, p.n, p.m, p.ldx, 32, kBM, true);
    const CUtensorMap th = map_2d(wh, p.n, wc, p.ldw, p.half ? 64 : 32, brows, true, esz);
    const CUtensorMap tl = map_2d(wl, p.n, wc, p.ldw, p.half ? 64 : 32, brows, true, esz);
    const bool first = c0 == 0, last = c0 + sw >= p.wpad;
    if (p.half)
      launch_pair<kXW, true>(s, tx, th, tl, a, num_sms, first ? p.ev_pre : nullptr, last ? p.ev_post : nullptr);
    else
      launch_pair<kXW, false>(s, tx, th, tl, a, num_sms, first ? p.ev_pre : nullptr, last ? p.ev_post : nullptr);
  }
}

// Row chunks per 256-column tile so that tiles x chunks spreads evenly over the
// pairs; chunks are whole 128-row blocks (the fp16 U^T scale granularity).
index_t utx_pair_splits(index_t m, index_t n, int num_sms, index_t* rows_per_split) {
  const index_t ntiles = ceil_div(n, 2 * kBM);
  index_t chunks = ceil_div(8 * static_cast<index_t>(num_sms / 2), ntiles);  // ~8 items per pair
  const index_t cap = env_int("LPCA_UTX_CHUNK_ROWS", 0);  // A/B: cap the rows per chunk (L2 reuse of U^T)
  if (cap > 0 && ceil_div(m, chunks) > cap) chunks = ceil_div(m, cap);
  const index_t max_chunks = ceil_div(m, 4 * kUScaleRows);                   // >= 4 runs per item
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  const index_t rows = round_up(ceil_div(m, chunks), kUScaleRows);  // chunks start on U^T scale blocks
  chunks = ceil_div(m, rows);
  *rows_per_split = rows;
  return chunks;
}

void launch_utx_pair(cudaStream_t s, const UtxPairArgs& p, int num_sms) {
  const index_t npad = round_up(p.l, 16);
  if (p.l < 1 || p.n < 1) throw Error(kInternal, "utx_pair: unsupported shape");
  if (p.ldx % 4 || (p.half ? p.ldt % 8 : p.ldt % 4))
    throw Error(kInternal, "utx_pair: leading dimensions must be 16-byte multiples");
  if (p.half && !p.uinv) throw Error(kInternal, "utx_pair: fp16 encoding needs the U^T scales");
  index_t rows = 0;
  const index_t chunks = utx_pair_splits(p.m, p.n, num_sms, &rows);
  const int esz = p.half ? 2 : 4;
  const int sw = slice_width(npad, true);
  for (index_t c0 = 0; c0 < npad; c0 += sw) {
    const int wc = static_cast<int>(npad - c0 < sw ? npad - c0 : sw);
    PairArgs a{};
    a.m = static_cast<int>(p.m);
    a.n = static_cast<int>(p.n);
    a.npad = wc;
    a.chunk_rows = static_cast<int>(rows);
    a.items = static_cast<int>(ceil_div(p.n, 2 * kBM) * chunks);
    a.run_stages = static_cast<int>(kUScaleRows / 64);  // fp16: one run per block of U^T scales
    a.scan = p.half && !p.xmax_in;
    a.xmax_in = p.xmax_in;
    a.uinv_in = p.uinv ? p.uinv + c0 : nullptr;
    a.uinv_ld = static_cast<int>(npad);
    a.part = p.part + c0;
    const index_t lc = p.l - c0;
    a.l = static_cast<int>(lc < wc ? lc : wc);
    a.l_ld = static_cast<int>(p.l);
    const uint32_t brows = static_cast<uint32_t>(wc / 2);
    const char* uh = static_cast<const char*>(p.u_hi) + c0 * p.ldt * esz;
    const char* ul = static_cast<const char*>(p.u_lo) + c0 * p.ldt * esz;
    const bool first = c0 == 0, last = c0 + sw >= npad;
    if (p.half) {
      const CUtensorMap tx = map_2d(p.x, p.n, p.m, p.ldx, kBM, 64, false);
      const CUtensorMap th = map_2d(uh, p.m, wc, p.ldt, 64, brows, true, 2);
      const CUtensorMap tl = map_2d(ul, p.m, wc, p.ldt, 64, brows, true, 2);
      launch_pair<kXTU, true>(s, tx, th, tl, a, num_sms, first ? p.ev_pre : nullptr, last ? p.ev_post : nullptr);
    } else {
      const CUtensorMap tx = map_2d(p.x, p.n, p.m, p.ldx, kBM, 32, false);
      const CUtensorMap th = map_2d(uh, p.m, wc, p.ldt, 32, brows, true);
      const CUtensorMap tl = map_2d(ul, p.m, wc, p.ldt, 32, brows, true);
      launch_pair<kXTU, false>(s, tx, th, tl, a, num_sms, first ? p.ev_pre : nullptr, last ? p.ev_post : nullptr);
    }
  }
}

void launch_xw_tc_planes(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx,
                         const float* w_hi, const float* w_lo, index_t wpad, index_t ldw, float* out,
                         index_t ldo, index_t wstore, float* out_hi, float* out_lo, index_t ldh,
                         int num_sms) {
  if (m <= 0) return;
  if (pair_mode()) {
    XwPairArgs p{};
    p.x = x;
    p.m = m;
    p.n = n;
    p.ldx = ldx;
    p.w_hi = w_hi;
    p.w_lo = w_lo;
    p.wpad = wpad;
    p.ldw = ldw;
    p.out = out;
    p.ldo = ldo;
    p.wstore = wstore;
    p.out_hi = out_hi;
    p.out_lo = out_lo;
    p.ldh = ldh;
    launch_xw_pair(s, p, num_sms);
    return;
  }
  TcArgs a{};
  if (!tc_xw_supported(n, wpad) || !plan_tmem(static_cast<int>(wpad), a))
    throw Error(kInternal, "xw_tc: unsupported shape");
  if (ldx % 4 || ldw % 4 || (out_hi && ldh % 4))
    throw Error(kInternal, "xw_tc: leading dimensions must be multiples of 4 floats");
  const CUtensorMap tx = map_2d(x, n, m, ldx, 32, kBM, true);
  const CUtensorMap th = map_2d(w_hi, n, wpad, ldw, 32, static_cast<uint32_t>(wpad), true);
  const CUtensorMap tl = map_2d(w_lo, n, wpad, ldw, 32, static_cast<uint32_t>(wpad), true);
  a.m = static_cast<int>(m);
  a.n = static_cast<int>(n);
  a.npad = static_cast<int>(wpad);
  a.items = static_cast<int>(ceil_div(m, kBM));
  a.chunks = 1;
  a.wstore = static_cast<int>(wstore);
  a.out = out;
  a.ldo = static_cast<int>(ldo);
  a.out_hi = out_hi;
  a.out_lo = out_lo;
  a.ldh = static_cast<int>(ldh);
  launch<kXW>(s, tx, th, tl, a, a.items < num_sms ? a.items : num_sms);
}

void launch_xw_tc(cudaStream_t s, const float* x, index_t m, index_t n, index_t ldx, const float* w_hi,
                  const float* w_lo, index_t wpad, index_t ldw, float* out, index_t ldo, int num_sms) {
  launch_xw_tc_planes(s, x, m, n, ldx, w_hi, w_lo, wpad, ldw, out, ldo, wpad, nullptr, nullptr, 0, num_sms);
}

// Row chunks per n tile so that tiles x chunks spreads evenly over the CTAs.
index_t utx_tc_splits(index_t m, index_t l, index_t n, int num_sms, index_t* rows_per_split) {
  (void)l;
  if (pair_mode()) return utx_pair_splits(m, n, num_sms, rows_per_split);
  const index_t ntiles = ceil_div(n, kBM);
  index_t chunks = ceil_div(8 * static_cast<index_t>(num_sms), ntiles);  // ~8 items per CTA
  const index_t max_chunks = ceil_div(m, 4 * kRunStages * kBK);          // >= 4 runs per item
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  const index_t rows = round_up(ceil_div(m, chunks), kBK);
  chunks = ceil_div(m, rows);
  *rows_per_split = rows;
  return chunks;
}

void launch_utx_tc_planes(cudaStream_t s, const float* ut_hi, const float* ut_lo, index_t ldt, const float* x,
                          index_t ldx, index_t m, index_t l, index_t n, double* part, int num_sms) {
  if (pair_mode()) {
    UtxPairArgs p{};
    p.u_hi = ut_hi;
    p.u_lo = ut_lo;
    p.ldt = ldt;
    p.x = x;
    p.ldx = ldx;
    p.m = m;
    p.l = l;
    p.n = n;
    p.part = part;
    launch_utx_pair(s, p, num_sms);
    return;
  }
  TcArgs a{};
  const index_t npad = round_up(l, 16);
  if (!tc_utx_supported(l, n) || !plan_tmem(static_cast<int>(npad), a))
    throw Error(kInternal, "utx_tc: unsupported shape");
  if (ldt % 4 || ldx % 4) throw Error(kInternal, "utx_tc: leading dimensions must be multiples of 4 floats");
  index_t rows = 0;
  const index_t chunks = utx_tc_splits(m, l, n, num_sms, &rows);
  a.m = static_cast<int>(m);
  a.n = static_cast<int>(n);
  a.npad = static_cast<int>(npad);
  a.chunks = static_cast<int>(chunks);
  a.chunk_rows = static_cast<int>(rows);
  a.items = static_cast<int>(ceil_div(n, kBM) * chunks);
  a.part = part;
  a.l = static_cast<int>(l);
  const CUtensorMap tx = map_2d(x, n, m, ldx, kBM, kBK, false);
  const CUtensorMap th = map_2d(ut_hi, m, npad, ldt, 32, static_cast<uint32_t>(npad), true);
  const CUtensorMap tl = map_2d(ut_lo, m, npad, ldt, 32, static_cast<uint32_t>(npad), true);
  launch<kXTU>(s, tx, th, tl, a, a.items < num_sms ? a.items : num_sms);
}

void launch_utx_tc(cudaStream_t, const float*, index_t, const float*, index_t, index_t, index_t, index_t,
                   index_t, double*, int) {
  throw Error(kInternal, "use launch_utx_tc_planes (U^T arrives as tf32 hi/lo planes)");
}

}  // namespace lpca

#ifdef LPCA_PAIR_PROF
extern "C" void lpca_debug_pair_prof(unsigned long long* out32, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out32, lpca::g_pair_prof, sizeof(unsigned long long) * 32);
  if (reset) {
    static const unsigned long long zero[32] = {};
    cudaMemcpyToSymbol(lpca::g_pair_prof, zero, sizeof(zero));
  }
}
#endif
