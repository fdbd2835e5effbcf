// 2-SM (cta_group::2) pass kernels: X W and X^T U with the 3-term split
//   a*b ~= a_hi*b_hi + a_lo*b_hi + a_hi*b_lo
// in one of two operand encodings:
//   kHalf = false : tf32 hi/lo (kind::tf32, K = 32 per stage). Needs no scale;
//                   the kernel-level exports (lpca_sketch_f32 / lpca_gemm_t_f32)
//                   and SPCA's Q^T X run this way.
//   kHalf = true  : fp16 hi/lo of power-of-two scaled operands (kind::f16,
//                   K = 64 per stage, twice the tf32 MMA rate, half the TMEM
//                   A traffic per K): every pass of Lazy SPCA. X rows are
//                   scaled per (row, run; 1024 deep) from the run's first stage
//                   (sketch, transform; a flagged run redoes the pass with each
//                   run scanned first) or by one s_x = 2^(14 - floor(log2
//                   max|X|)) from the max the sketch recorded (power step, F);
//                   the small operand per column (W planes) or per column and
//                   256-row block (U^T planes, written by the X W epilogue).
//                   hi = fp16_rn(a s), lo = fp16_rn(a s - hi): with every
//                   scaled value in [2^-14, 2^15] the split keeps 22 bits
//                   (tf32 hi/lo keeps 20); values more than 2^18 below their
//                   scale's maximum lose relative precision gradually.
// Scales are exact powers of two; results are unscaled per run (X^T U) or at
// the final store (X W) before they leave the kernel.
//
// Why pairs: at the fit's widths (N = 112..224) every stage of the 1-SM kernel
// moves the B planes through L2, TMA and shared memory for 12 MMAs; a CTA pair
// issues M = 256 MMAs with each CTA holding its own 128 rows of A (in TMEM) and
// half of B (N/2 rows) — per SM, B traffic halves.
//
// Protocol (leader = cluster rank 0 issues every MMA):
//   full_x[s]   local   : TMA of this CTA's X tile landed (converter waits)
//   full_b[s]   leader  : both B halves landed (2-SM TMA form signals rank 0)
//   conv[a]     leader  : 8 converter warps (4 per CTA) wrote their A slot
//   aempty[a]   each    : multicast commit, MMAs done with A slot a
//   empty[s]    each    : multicast commit, MMAs done with smem stage s
//   tfull[b]    each    : multicast commit, run accumulated in run buffer b
//   tempty[b]   leader  : 8 epilogue warps drained run buffer b
// Remote arrivals use mapa + mbarrier.arrive on the shared::cluster address;
// waits are the usual cta-scoped try_wait loops (as CUTLASS's cluster barriers).
//
// Included by gemm_tc.cu inside its anonymous namespace (shares kBM, kThreads,
// kXW/kXTU and the tc:: helpers). Work items: XW 256-row tiles (128 per CTA);
// XTU 256-column tiles x row chunks.
#pragma once
#include <cuda_fp16.h>

// Per-run A-row scales in flight (scan mode): the converters write run R's
// scales before converting it, when the epilogue may still be folding run
// R - 4 (MMA up to nrb = 2 runs ahead of the epilogue, converters up to two
// stages = one run ahead of the MMA, plus the run being scanned): a ring of 8.
constexpr int kRscRing = 8;

struct PairArgs {
  int m, n;          // X is m x n
  int npad;          // UMMA N (multiple of 16); each CTA holds npad / 2 rows of B
  int stages, aslots, nrb, run_stages;
  int half_slots;  // fp16 A ring granularity: 0 = full-stage slots (64 columns, K = 64), 2 = half-stage
                   // slots (32 columns, K = 32), 4 = quarter-stage slots (16 columns, K = 16)
  uint32_t tmem_cols;
  int items;
  int chunk_rows;    // XTU: rows per chunk (multiple of 128)
  // fp16 A scale: scan = 1 gives every (row, run) its own power of two from the
  // run's values (scanned in shared memory first); scan = 2 takes it from the
  // run's first stage with 16x headroom and flags (*ovf) any later stage that
  // would overflow fp16 or sit 2^8 below the range (the caller then reruns with
  // scan = 1); scan = 0 uses one scale for all of X from max|X| = *xmax_in
  // (bits) or xmax_val
  int scan;
  int* ovf;
  const int* wlo_nz;  // X W: nonzero when W's lo plane has a nonzero entry (null: assume it does)
  const uint32_t* xmax_in;
  float xmax_val;
  // X W: accumulate max|X| bits of the data actually read here (nullable)
  uint32_t* xmax_out;
  // X W, fp16: inverse column scales of the W planes (npad)
  const float* winv;
  // X W outputs
  int wstore;
  float* out;        // plain fp32 row-major (nullable)
  int ldo;
  float* out_hi;     // tf32 planes of OUT^T [npad][ldh] (nullable)
  float* out_lo;
  __half* uh;        // fp16 planes of OUT^T [npad][ldh] with block scales (nullable)
  __half* ul;
  float* uinv;       // [ceil(m/256)][npad] inverse block scales of uh/ul
  int ldh;
  // X^T U: U^T block inverse scales (fp16), partial output part[chunk][j * l + r]
  const float* uinv_in;
  double* part;
  int l;      // X^T U: columns r < l of the part rows are stored ...
  int l_ld;   // ... with row stride l_ld (N-split launches write column slices)
  int uinv_ld;  // row stride of the [block][c] inverse scales (uinv / uinv_in)
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  // default .release.cta semantics (as CUTLASS's ClusterBarrier::arrive): the
  // .cluster-scoped release compiles to MEMBAR.ALL.GPU + ERRBAR per arrival and
  // made each pipeline stage cost ~1 us. TMEM ordering comes from the tcgen05
  // fences around the barrier, not from the arrive's memory scope.
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// B half-tile load: lands in this CTA's smem, completes bytes on the leader's barrier.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
// Arrives on `bar` (same offset) in both CTAs of the pair once the issued MMAs complete.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// One stage of the 3-term split as 12 M = 256 pair MMAs, A from TMEM of both
// CTAs: four K-steps (tf32: K = 8, fp16: K = 16), each 8 TMEM columns of A and
// 32 B of the B rows (descriptor +2).
#define LPCA_PAIR_STAGE(KIND)                                                                              \
  "{\n .reg .pred p, t, bl;\n setp.ne.b32 p, %6, 0;\n setp.eq.u32 t, %7, %7;\n setp.ne.b32 bl, %7, 0;\n"                                \
  " .reg .b32 ah, al;\n .reg .b64 dh, dl;\n"                                                              \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [%1], %3, %5, p;\n"                                     \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [%2], %3, %5, t;\n"                                     \
  " @bl tcgen05.mma.cta_group::2.kind::" KIND " [%0], [%1], %4, %5, t;\n"                                     \
  " add.u32 ah, %1, 8;\n add.u32 al, %2, 8;\n add.u64 dh, %3, 2;\n add.u64 dl, %4, 2;\n"                   \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dh, %5, t;\n"                                     \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [al], dh, %5, t;\n"                                     \
  " @bl tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dl, %5, t;\n"                                     \
  " add.u32 ah, %1, 16;\n add.u32 al, %2, 16;\n add.u64 dh, %3, 4;\n add.u64 dl, %4, 4;\n"                 \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dh, %5, t;\n"                                     \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [al], dh, %5, t;\n"                                     \
  " @bl tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dl, %5, t;\n"                                     \
  " add.u32 ah, %1, 24;\n add.u32 al, %2, 24;\n add.u64 dh, %3, 6;\n add.u64 dl, %4, 6;\n"                 \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dh, %5, t;\n"                                     \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [al], dh, %5, t;\n"                                     \
  " @bl tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dl, %5, t;\n"                                     \
  "}"

// Half a stage (K = 32, fp16): 6 MMAs from a 32-column half slot (hi 16, lo 16).
#define LPCA_PAIR_HALF(KIND)                                                                               \
  "{\n .reg .pred p, t, bl;\n setp.ne.b32 p, %6, 0;\n setp.eq.u32 t, %7, %7;\n setp.ne.b32 bl, %7, 0;\n"                                \
  " .reg .b32 ah, al;\n .reg .b64 dh, dl;\n"                                                              \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [%1], %3, %5, p;\n"                                     \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [%2], %3, %5, t;\n"                                     \
  " @bl tcgen05.mma.cta_group::2.kind::" KIND " [%0], [%1], %4, %5, t;\n"                                     \
  " add.u32 ah, %1, 8;\n add.u32 al, %2, 8;\n add.u64 dh, %3, 2;\n add.u64 dl, %4, 2;\n"                   \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dh, %5, t;\n"                                     \
  " tcgen05.mma.cta_group::2.kind::" KIND " [%0], [al], dh, %5, t;\n"                                     \
  " @bl tcgen05.mma.cta_group::2.kind::" KIND " [%0], [ah], dl, %5, t;\n"                                     \
  "}"
__device__ __forceinline__ void mma_half_pair(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh, uint64_t bl,
                                              uint32_t idesc, uint32_t acc_first, uint32_t blo) {
  asm volatile(LPCA_PAIR_HALF("f16")::"r"(d), "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(idesc), "r"(acc_first),
               "r"(blo)
               : "memory");
}
#undef LPCA_PAIR_HALF

// A quarter stage (K = 16, fp16): 3 MMAs from a 16-column quarter slot (hi 8, lo 8).
__device__ __forceinline__ void mma_quarter_pair(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh, uint64_t bl,
                                                 uint32_t idesc, uint32_t acc_first, uint32_t blo) {
  asm volatile(
      "{\n .reg .pred p, t, bl;\n setp.ne.b32 p, %6, 0;\n setp.eq.u32 t, %7, %7;\n setp.ne.b32 bl, %7, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %3, %5, p;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], [%2], %3, %5, t;\n"
      " @bl tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %4, %5, t;\n"
      "}" ::"r"(d),
      "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(idesc), "r"(acc_first), "r"(blo)
      : "memory");
}

template <bool kHalf>
__device__ __forceinline__ void mma_stage_pair(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh, uint64_t bl,
                                               uint32_t idesc, uint32_t acc_first, uint32_t blo) {
  if constexpr (kHalf)
    asm volatile(LPCA_PAIR_STAGE("f16")::"r"(d), "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(idesc),
                 "r"(acc_first), "r"(blo)
                 : "memory");
  else
    asm volatile(LPCA_PAIR_STAGE("tf32")::"r"(d), "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(idesc),
                 "r"(acc_first), "r"(blo)
                 : "memory");
}
#undef LPCA_PAIR_STAGE

// Instruction descriptor, kind::f16 with fp16 A/B and fp32 accumulation.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// s = 2^(14 - floor(log2 mx)) so that |a| s < 2^15 for |a| <= mx (1 for mx = 0,
// inf or NaN), built from the exponent bits (subnormal mx counts as 2^-126).
__device__ __forceinline__ float pow2_scale_for(float mx) {
  if (!(mx > 0.0f) || isinf(mx)) return 1.0f;
  int e = static_cast<int>((__float_as_uint(mx) >> 23) & 0xffu) - 127;
  e = e < -126 ? -126 : e;
  int t = 14 - e;
  t = t > 126 ? 126 : (t < -126 ? -126 : t);
  return __uint_as_float(static_cast<uint32_t>(t + 127) << 23);
}

// Scale for X rows: 1 (no multiply in the converters) whenever the row's max
// (times the headroom) already sits inside fp16's range with a normal hi term
// (2^-3 <= mx, headroom * mx < 2^15); otherwise the power of two that puts it at
// [2^14, 2^15). With scale 1, values far below the max keep an absolute error
// under 2^-25 (subnormal lo), below the max element's own 2^-22 relative error.
__device__ __forceinline__ float pow2_scale_x(float mx, float headroom) {
  if (mx >= 0.125f && headroom * mx < 32768.0f) return 1.0f;
  return pow2_scale_for(headroom * mx);
}

// Max over the warp's 32 lanes of each of x[0..15] in 16 shuffles (halving
// butterfly). Lane L ends with the max of column
//   ((L >> 4) & 1) * 8 + ((L >> 3) & 1) * 4 + ((L >> 2) & 1) * 2 + ((L >> 1) & 1).
__device__ __forceinline__ float warp_max16(const float (&x)[16], int lane) {
  const bool u4 = lane & 16, u3 = lane & 8, u2 = lane & 4, u1 = lane & 2;
  float y8[8], y4[4], y2[2];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    y8[j] = fmaxf(u4 ? x[8 + j] : x[j], __shfl_xor_sync(0xffffffffu, u4 ? x[j] : x[8 + j], 16));
#pragma unroll
  for (int j = 0; j < 4; ++j)
    y4[j] = fmaxf(u3 ? y8[4 + j] : y8[j], __shfl_xor_sync(0xffffffffu, u3 ? y8[j] : y8[4 + j], 8));
#pragma unroll
  for (int j = 0; j < 2; ++j)
    y2[j] = fmaxf(u2 ? y4[2 + j] : y4[j], __shfl_xor_sync(0xffffffffu, u2 ? y4[j] : y4[2 + j], 4));
  float y = fmaxf(u1 ? y2[1] : y2[0], __shfl_xor_sync(0xffffffffu, u1 ? y2[0] : y2[1], 2));
  return fmaxf(y, __shfl_xor_sync(0xffffffffu, y, 1));
}
__device__ __forceinline__ int warp_max16_col(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Splits 32 consecutive-K values (already scaled) into 16 packed hi and 16 packed lo columns.
__device__ __forceinline__ void split_f16_32(const float (&v)[32], float (&hi)[16], float (&lo)[16]) {
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const __half2 h = __floats2half2_rn(v[2 * c], v[2 * c + 1]);
    const float2 hf = __half22float2(h);
    hi[c] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&h));
    lo[c] = __uint_as_float(pack_h2(v[2 * c] - hf.x, v[2 * c + 1] - hf.y));
  }
}

// Splits 16 consecutive-K values (already scaled) into 8 packed hi and 8 packed lo columns.
__device__ __forceinline__ void split_f16_16(const float* v, float (&hi)[8], float (&lo)[8]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const __half2 h = __floats2half2_rn(v[2 * c], v[2 * c + 1]);
    const float2 hf = __half22float2(h);
    hi[c] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&h));
    lo[c] = __uint_as_float(pack_h2(v[2 * c] - hf.x, v[2 * c + 1] - hf.y));
  }
}

// The items a pair works through. X W: the consecutive 256-row items of one
// kUScaleRows block of U^T scales back to back, so the block's later items can
// settle the block's scales; X^T U: every npairs-th item. -1 when done.
constexpr int kItemsPerBlock = static_cast<int>(kUScaleRows) / 256;
template <int kMode>
__device__ __forceinline__ int pair_item(int pair, int npairs, int it, int items) {
  if (kMode == kXW) {
    const int item = kItemsPerBlock * (pair + (it / kItemsPerBlock) * npairs) + it % kItemsPerBlock;
    return item < items ? item : -1;
  }
  const int item = pair + it * npairs;
  return item < items ? item : -1;
}

template <int kMode>
__device__ __forceinline__ void pair_item_coords(const PairArgs& a, int item, int& t0, int& k0, int& k1) {
  if (kMode == kXW) {
    t0 = item * 2 * kBM;
    k0 = 0;
    k1 = a.n;
  } else {
    // chunk-major: pairs running together share row chunks (U^T planes stay in L2)
    const int ntiles = (a.n + 2 * kBM - 1) / (2 * kBM);
    const int nt = item % ntiles, ch = item / ntiles;
    t0 = nt * 2 * kBM;
    k0 = ch * a.chunk_rows;
    k1 = min(a.m, k0 + a.chunk_rows);
  }
}

// Epilogue warps (kEpi). Wide X W slices (one TMEM run buffer): two per TMEM
// lane quadrant, each folding and writing half of the accumulator's columns (the
// fold releases the run buffer twice as soon: the MMA's wait for it fell from
// 15% to 6% at configs[2]). Otherwise one per quadrant: X^T U's converters need
// the registers (at 448 threads ptxas caps them at 128 and the column-wise
// transposing loads spill), and narrow slices have two run buffers anyway.
// Converter warps: one per TMEM lane quadrant, or (LPCA_TC_CONV, wide fp16 X W
// slices with quarter A slots) two, each converting one 32-column half of every
// stage, so one warp's split overlaps the other's TMEM-store and hand-off
// latency. The MMA's wait for converted A falls from 39% to 20% of its time at
// configs[2], but the power-capped passes are no faster, so one is the default.
constexpr int pair_threads(int conv, int epi) {
  return 32 * (2 + conv + epi);  // TMA, MMA, converters, the epilogue
}
constexpr int kMaxEpiWarps = 8;
template <int kEpi>
__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpi) : "memory");
}

#ifdef LPCA_PAIR_PROF  // role timers (tools/pair_prof.py): cycles summed over CTAs
__device__ unsigned long long g_pair_prof[2][16];  // [mode][counter]
#define PP_T0() const long long pp_t0_ = clock64()
#define PP_ADD(k) \
  if (lane == 0) pp[k] += clock64() - pp_t0_
#else
#define PP_T0()
#define PP_ADD(k)
#endif

template <int kMode, bool kHalf, int kEpi, int kConv = 4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair_threads(kConv, kEpi), 1)
    tc2_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmbh,
               const __grid_constant__ CUtensorMap tmbl, PairArgs a) {
  constexpr int BK = kHalf ? 64 : 32;  // K per stage (one 128 B swizzle row of B)
  constexpr int kEpiWarps = kEpi;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by pointer arithmetic on the shared array (an integer round
  // trip would lose the address space and turn every access generic)
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  const int S = a.stages, AS = a.aslots;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  constexpr uint32_t x_bytes = kBM * BK * 4;                              // this CTA's 128 A rows (fp32)
  const uint32_t bh_bytes = static_cast<uint32_t>(a.npad / 2) * 128;     // this CTA's half of one B plane
  const uint32_t stage_bytes = x_bytes + 2 * bh_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* full_x = bars;
  uint64_t* full_b = full_x + S;
  uint64_t* empty = full_b + S;
  uint64_t* conv = empty + S;
  uint64_t* aempty = conv + AS;
  uint64_t* tfull = aempty + AS;
  uint64_t* tempty = tfull + 2;
  uint64_t* xch = tempty + 2;  // [2] U^T block-maximum exchange with the peer (XW fp16 planes)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xch + 2);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [kEpiWarps][npad] epilogue block maxima / run scales
  float* rsc = red + (kMaxEpiWarps + 1) * a.npad;  // after red + gsc [npad]: [kRscRing runs][128] inverse A-row scales
  float* xbuf = rsc + kRscRing * kBM;  // [2][npad] the peer's column maxima (written by the peer)
  float* xrow = xbuf + 2 * a.npad;     // [2][128] row maxima of the two converter halves (8 converters)
  static_assert(kConv == 4 || (kConv == 8 && kMode == kXW && kHalf), "8 converters: fp16 X W only");

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t a_col0 = static_cast<uint32_t>((a.nrb + 1) * a.npad);
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int run_k = a.run_stages * BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_x[s], 1);
      mbar_init(&full_b[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(&conv[s], 8);
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kEpiWarps);
      mbar_init(&xch[b], 1);
    }
    fence_barrier_init();
    tma_prefetch(&tmx);
    tma_prefetch(&tmbh);
    tma_prefetch(&tmbl);
  }
  if (warp == 1) tmem_alloc2(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrival
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  float xs = 1.0f;  // s_x (fp16 encoding)
  if (kHalf) xs = pow2_scale_x(a.xmax_in ? __uint_as_float(*a.xmax_in) : a.xmax_val, 1.0f);

#ifdef LPCA_PAIR_PROF
  long long pp[16] = {};
  const long long pp_start = clock64();
#endif
  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int brow = static_cast<int>(rank) * (a.npad / 2);
      for (int it = 0, item; (item = pair_item<kMode>(pair, npairs, it, a.items)) >= 0; ++it) {
        int t0, k0, k1;
        pair_item_coords<kMode>(a, item, t0, k0, k1);
        const int mine = t0 + static_cast<int>(rank) * kBM;
        for (int k = k0; k < k1; k += BK) {
          {
            PP_T0();
            mbar_wait(&empty[stage], phase ^ 1, 1);
            PP_ADD(0);
          }
          uint8_t* st = smem + stage * stage_bytes;
          mbar_expect_tx(&full_x[stage], x_bytes);
          if (kMode == kXW) {
            tma_load_2d(st, &tmx, &full_x[stage], k, mine);  // [128 rows][32 fp32] SW128 sub-tiles
            if (kHalf) tma_load_2d(st + 16384, &tmx, &full_x[stage], k + 32, mine);
          } else {
            tma_load_2d(st, &tmx, &full_x[stage], mine, k);  // [BK rows][128 cols]
          }
          if (leader) mbar_expect_tx(&full_b[stage], 4 * bh_bytes);  // both halves, both planes
          tma_load_2d_pair(st + x_bytes, &tmbh, &full_b[stage], k, brow);
          tma_load_2d_pair(st + x_bytes + bh_bytes, &tmbl, &full_b[stage], k, brow);
          ring_advance(stage, phase, S);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only, whole warp) ----------------
    if (leader) {
      const uint32_t idesc = kHalf ? idesc_f16(2 * kBM, a.npad) : idesc_tf32(2 * kBM, a.npad, 0, 0);
      // B's lo plane all zero (W exact in fp16, e.g. a very sparse Omega): the
      // a_hi b_lo products add exact zeros and are skipped
      const uint32_t blo = (kMode == kXW && a.wlo_nz && *a.wlo_nz == 0) ? 0u : 1u;
      const uint64_t desc0 = sw128_desc(smem_u32(smem) + x_bytes, 16, 1024);
      int stage = 0, aslot = 0, rc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int it = 0, item; (item = pair_item<kMode>(pair, npairs, it, a.items)) >= 0; ++it) {
        int t0, k0, k1;
        pair_item_coords<kMode>(a, item, t0, k0, k1);
        for (int q0 = k0; q0 < k1; q0 += run_k, ++rc) {
          const int b = rc % a.nrb;
          {
            PP_T0();
            mbar_wait(&tempty[b], ((rc / a.nrb) & 1) ^ 1, 2);
            PP_ADD(2);
          }
          tc_fence_after();
          const uint32_t d = tmem_base + static_cast<uint32_t>(b * a.npad);
          const int q1 = min(k1, q0 + run_k);
          for (int k = q0; k < q1; k += BK) {
            {
              PP_T0();
              mbar_wait(&conv[aslot], aphase, 3);
              PP_ADD(3);
            }
            {
              PP_T0();
              mbar_wait(&full_b[stage], phase, 3);
              PP_ADD(4);
            }
            tc_fence_after();
            const uint64_t bh = desc0 + static_cast<uint64_t>((stage * stage_bytes) >> 4);
            const uint64_t bl = bh + static_cast<uint64_t>(bh_bytes >> 4);
            if (kHalf && a.half_slots == 4) {
              // four quarter slots per stage (K = 16 each): a freed quarter is
              // refilled while the MMAs read the other three (B rows advance 2
              // descriptor units = 32 B per quarter)
              for (int hh = 0; hh < 4; ++hh) {
                if (hh > 0) {
                  PP_T0();
                  mbar_wait(&conv[aslot], aphase, 3);
                  PP_ADD(3);
                  tc_fence_after();
                }
                const uint32_t at = tmem_base + a_col0 + static_cast<uint32_t>(aslot * 16);
                if (elect_one()) {
                  mma_quarter_pair(d, at, at + 8, bh + 2 * hh, bl + 2 * hh, idesc, (k != q0 || hh) ? 1u : 0u, blo);
                  if (hh == 3) mma_commit_pair(&empty[stage]);
                  mma_commit_pair(&aempty[aslot]);
                }
                __syncwarp();
                ring_advance(aslot, aphase, AS);
              }
              ring_advance(stage, phase, S);
              continue;
            }
            if (kHalf && a.half_slots) {
              // two half slots per stage: the converters fill one while the
              // MMAs read the other (B rows advance 4 descriptor units per half)
              for (int hh = 0; hh < 2; ++hh) {
                if (hh == 1) {
                  PP_T0();
                  mbar_wait(&conv[aslot], aphase, 3);
                  PP_ADD(3);
                  tc_fence_after();
                }
                const uint32_t at = tmem_base + a_col0 + static_cast<uint32_t>(aslot * 32);
                if (elect_one()) {
                  mma_half_pair(d, at, at + 16, bh + 4 * hh, bl + 4 * hh, idesc, (k != q0 || hh) ? 1u : 0u, blo);
                  if (hh == 1) mma_commit_pair(&empty[stage]);
                  mma_commit_pair(&aempty[aslot]);
                }
                __syncwarp();
                ring_advance(aslot, aphase, AS);
              }
              ring_advance(stage, phase, S);
              continue;
            }
            const uint32_t at = tmem_base + a_col0 + static_cast<uint32_t>(aslot * 64);
            if (elect_one()) {
              mma_stage_pair<kHalf>(d, at, at + 32, bh, bl, idesc, k != q0 ? 1u : 0u, blo);
              mma_commit_pair(&empty[stage]);
              mma_commit_pair(&aempty[aslot]);
            }
            __syncwarp();
            ring_advance(stage, phase, S);
            ring_advance(aslot, aphase, AS);
          }
          if (elect_one()) mma_commit_pair(&tfull[b]);
          __syncwarp();
        }
      }
    }
  } else if (warp < 2 + kConv) {
    // ---------------- converters (both CTAs): smem X -> own TMEM A ----------------
    const int q = warp & 3;
    const int hsel = kConv == 8 ? (warp - 2) >> 2 : 0;  // 8 converters: this warp's 32-column half
    // 8 converters: a row's maximum over both halves (the two warps of a quadrant)
    auto row_max_both = [&](float mine) {
      xrow[hsel * kBM + q * 32 + lane] = mine;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
      const float m = fmaxf(xrow[q * 32 + lane], xrow[kBM + q * 32 + lane]);
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
      return m;
    };
    const int i = q * 32 + lane;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    float xmax = 0.0f;
    int stage = 0, aslot = 0, rc = 0;
    uint32_t phase = 0, aphase = 0;
    auto load_row = [&](const uint8_t* xt, int h, float (&v)[32]) {
      if (kMode == kXW) {
        // row i of a 128 B-swizzled [128][32] sub-tile: 16 B chunk c at (c ^ (i & 7))
        const uint8_t* sub = xt + h * 16384;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 f = *reinterpret_cast<const float4*>(sub + i * 128 + ((c ^ (i & 7)) << 4));
          v[4 * c] = f.x;
          v[4 * c + 1] = f.y;
          v[4 * c + 2] = f.z;
          v[4 * c + 3] = f.w;
        }
      } else {
        // column i of a plain [BK][128] tile, rows 32h..32h+31
        const float* raw = reinterpret_cast<const float*>(xt) + h * 32 * kBM;
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) v[kk] = raw[kk * kBM + i];
      }
    };
    auto absmax32k = [](const float (&v)[32]) {  // the same tree, keeping v
      float t[16];
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) t[kk] = fmaxf(fabsf(v[kk]), fabsf(v[kk + 16]));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) t[kk] = fmaxf(t[kk], t[kk + 8]);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) t[kk] = fmaxf(t[kk], t[kk + 4]);
      return fmaxf(fmaxf(t[0], t[1]), fmaxf(t[2], t[3]));
    };
    bool ovf = false;
    auto absmax32 = [](float (&v)[32]) {  // tree (a serial max chain is latency-bound); clobbers v
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) v[kk] = fmaxf(fabsf(v[kk]), fabsf(v[kk + 16]));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) v[kk] = fmaxf(v[kk], v[kk + 8]);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) v[kk] = fmaxf(v[kk], v[kk + 4]);
      return fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
    };
    for (int it = 0, item; (item = pair_item<kMode>(pair, npairs, it, a.items)) >= 0; ++it) {
      int t0, k0, k1;
      pair_item_coords<kMode>(a, item, t0, k0, k1);
      for (int q0 = k0; q0 < k1; q0 += run_k, ++rc) {
        const int nst = (min(k1, q0 + run_k) - q0 + BK - 1) / BK;
        float sx = xs;
        if (kHalf && a.scan == 1) {  // the run's stages are all resident (run_stages <= stages)
          float mx = 0.0f;
          int st = stage;
          uint32_t ph = phase;
          for (int j = 0; j < nst; ++j) {
            mbar_wait(&full_x[st], ph, 4);
            const uint8_t* xt = smem + st * stage_bytes;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (kConv == 8 && h != hsel) continue;
              float v[32];
              load_row(xt, h, v);
              mx = fmaxf(mx, absmax32(v));
            }
            ring_advance(st, ph, S);
          }
          xmax = fmaxf(xmax, mx);
          if (kConv == 8) mx = row_max_both(mx);
          sx = pow2_scale_x(mx, 1.0f);
          if (hsel == 0) rsc[(rc % kRscRing) * kBM + i] = __frcp_rn(sx);
        }
        for (int j = 0; j < nst; ++j) {
          if constexpr (kConv == 8) {
            // one 32-column half of the stage -> its two quarter slots
            mbar_wait(&full_x[stage], phase, 4);
            const uint8_t* xt = smem + stage * stage_bytes;
            float v[32];
            load_row(xt, hsel, v);
            if (a.scan == 2 || (a.xmax_out && a.scan == 0)) {
              const float mh = absmax32k(v);
              if (a.xmax_out) xmax = fmaxf(xmax, mh);
              if (a.scan == 2) {
                if (j == 0) {  // the run's scale: 16x headroom over its first stage (both halves)
                  sx = pow2_scale_x(row_max_both(mh), 16.0f);
                  if (hsel == 0) rsc[(rc % kRscRing) * kBM + i] = __frcp_rn(sx);
                } else if (mh * sx >= 32768.0f || (mh > 0.0f && mh * sx < 0.125f)) {
                  ovf = true;
                }
              }
            }
            if (__any_sync(0xffffffffu, sx != 1.0f)) {
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) v[kk] *= sx;
            }
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              if ((qq >> 1) == hsel) {
                float h8[8], l8[8];
                split_f16_16(v + 16 * (qq & 1), h8, l8);
                mbar_wait(&aempty[aslot], aphase ^ 1, 4);
                tc_fence_after();
                const uint32_t aq = lane_base + a_col0 + static_cast<uint32_t>(aslot * 16);
                tmem_st8(aq, h8);
                tmem_st8(aq + 8, l8);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&conv[aslot]), 0));
              }
              ring_advance(aslot, aphase, AS);
            }
            ring_advance(stage, phase, S);
            continue;
          }
          {
            PP_T0();
            mbar_wait(&full_x[stage], phase, 4);
            if (q == 0) PP_ADD(6);
          }
          {
            PP_T0();
            mbar_wait(&aempty[aslot], aphase ^ 1, 4);
            if (q == 0) PP_ADD(7);
          }
          tc_fence_after();
          const uint8_t* xt = smem + stage * stage_bytes;
          const uint32_t at =
              lane_base + a_col0 + static_cast<uint32_t>(aslot * (a.half_slots == 4 ? 16 : a.half_slots ? 32 : 64));
          if (kHalf) {
            float v0[32], v1[32];
#ifdef LPCA_PAIR_PROF
            long long pp_c0 = clock64();
#endif
            load_row(xt, 0, v0);
            load_row(xt, 1, v1);
#ifdef LPCA_PAIR_PROF
            if (v0[0] == 1.2345e-30f || v1[31] == 1.2345e-30f) pp_c0 = 0;
            if (q == 0 && lane == 0) pp[1] += clock64() - pp_c0;
            pp_c0 = clock64();
#endif
            if (a.scan == 2 || (kMode == kXW && a.xmax_out && a.scan == 0)) {
              const float mx = fmaxf(absmax32k(v0), absmax32k(v1));
              if (kMode == kXW && a.xmax_out) xmax = fmaxf(xmax, mx);
              if (a.scan == 2) {
                if (j == 0) {  // the run's scale: 16x headroom over its first stage
                  sx = pow2_scale_x(mx, 16.0f);
                  rsc[(rc % kRscRing) * kBM + i] = __frcp_rn(sx);
                } else if (mx * sx >= 32768.0f || (mx > 0.0f && mx * sx < 0.125f)) {
                  ovf = true;
                }
              }
            }
            if (__any_sync(0xffffffffu, sx != 1.0f)) {
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) {
                v0[kk] *= sx;
                v1[kk] *= sx;
              }
            }
            float hi[16], lo[16];
            if (a.half_slots == 4) {  // quarters 0..3 -> four consecutive slots (the first one is held)
#pragma unroll
              for (int qq = 0; qq < 4; ++qq) {
                float h8[8], l8[8];
                split_f16_16((qq < 2 ? v0 : v1) + 16 * (qq & 1), h8, l8);
                if (qq > 0) {
                  ring_advance(aslot, aphase, AS);
                  mbar_wait(&aempty[aslot], aphase ^ 1, 4);
                  tc_fence_after();
                }
                const uint32_t aq = lane_base + a_col0 + static_cast<uint32_t>(aslot * 16);
                tmem_st8(aq, h8);
                tmem_st8(aq + 8, l8);
                if (qq < 3) {
                  tmem_st_wait();
                  tc_fence_before();
                  __syncwarp();
                  if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&conv[aslot]), 0));
                }
              }
            } else if (a.half_slots) {  // half 0 -> this slot, then half 1 -> the next one
              split_f16_32(v0, hi, lo);
              tmem_st16(at, hi);
              tmem_st16(at + 16, lo);
              tmem_st_wait();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&conv[aslot]), 0));
              ring_advance(aslot, aphase, AS);
              mbar_wait(&aempty[aslot], aphase ^ 1, 4);
              tc_fence_after();
              const uint32_t at1 = lane_base + a_col0 + static_cast<uint32_t>(aslot * 32);
              split_f16_32(v1, hi, lo);
              tmem_st16(at1, hi);
              tmem_st16(at1 + 16, lo);
            } else {
              split_f16_32(v0, hi, lo);
              tmem_st16(at, hi);
              tmem_st16(at + 32, lo);
              split_f16_32(v1, hi, lo);
              tmem_st16(at + 16, hi);
              tmem_st16(at + 48, lo);
            }
#ifdef LPCA_PAIR_PROF
            if (q == 0 && lane == 0) pp[5] += clock64() - pp_c0;
#endif
          } else {
            float v[32];
            load_row(xt, 0, v);
            if (kMode == kXW && a.xmax_out && a.scan == 0) {
              float t[32];
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) t[kk] = v[kk];
              xmax = fmaxf(xmax, absmax32(t));
            }
            {
              float hi[32], lo[32];
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) {
                hi[kk] = tf32_trunc(v[kk]);
                lo[kk] = tf32_trunc(v[kk] - hi[kk]);
              }
              tmem_st32(at, hi);
              tmem_st32(at + 32, lo);
            }
          }
#ifdef LPCA_PAIR_PROF
          long long pp_w0 = clock64();
#endif
          tmem_st_wait();
#ifdef LPCA_PAIR_PROF
          if (q == 0 && lane == 0) pp[8] += clock64() - pp_w0;
          pp_w0 = clock64();
#endif
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&conv[aslot]), 0));
#ifdef LPCA_PAIR_PROF
          if (q == 0 && lane == 0) pp[10] += clock64() - pp_w0;
#endif
          ring_advance(stage, phase, S);
          ring_advance(aslot, aphase, AS);
        }
      }
    }
    if (kMode == kXW && a.xmax_out) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
      if (lane == 0) atomicMax(a.xmax_out, __float_as_uint(xmax));
    }
    if (kHalf && a.scan == 2 && __any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(a.ovf, 1);
  } else {
    // ---------------- epilogue (both CTAs, own 128 rows) ----------------
    const int q = warp & 3;                       // TMEM lane quadrant
    const int ew = warp - 2 - kConv;              // epilogue warp 0 .. kEpiWarps - 1
    const int nch16 = a.npad / 16;                // this warp's 16-column chunks: one half of them
    const int half = ew / 4;
    const int c_lo = kEpiWarps == 4 ? 0 : (half ? (nch16 + 1) / 2 : 0) * 16;
    const int c_hi = kEpiWarps == 4 ? a.npad : (half ? nch16 : (nch16 + 1) / 2) * 16;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t lacc = lane_base + static_cast<uint32_t>(a.nrb * a.npad);
    const float xinv = 1.0f / xs;
    int rc = 0;
    int xit = 0;  // planes16 items done (xch / xbuf parity)
    for (int it = 0, item; (item = pair_item<kMode>(pair, npairs, it, a.items)) >= 0; ++it) {
      int t0, k0, k1;
      pair_item_coords<kMode>(a, item, t0, k0, k1);
      const int runs = (k1 - k0 + run_k - 1) / run_k;
      const int row = t0 + static_cast<int>(rank) * kBM + q * 32 + lane;  // XW: X row; XTU: X column
      const bool to_planes16 = kMode == kXW && a.uh != nullptr;
      // X^T U, fp16: each run's rows form one 256-row block of U^T scales. The
      // next run's scales are fetched into registers while this run is folded
      // and staged in this warp's row of red[] (broadcast reads).
      float* runsc = red + ew * a.npad;
      float nxt[8];
      auto fetch_scales = [&](int r) {
        const float* src = a.uinv_in + static_cast<size_t>((k0 + r * run_k) / kUScaleRows) * a.uinv_ld;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = lane + 32 * j;
          nxt[j] = c < a.npad ? __ldg(src + c) : 0.0f;  // scaled when staged (no stall here)
        }
      };
      if (kMode == kXTU && kHalf) fetch_scales(0);
      for (int r = 0; r < runs; ++r, ++rc) {
        const int b = rc % a.nrb;
        if (kMode == kXTU && kHalf) {
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (lane + 32 * j < a.npad) runsc[lane + 32 * j] = nxt[j];
          __syncwarp();
          if (r + 1 < runs) fetch_scales(r + 1);
        }
        {
          PP_T0();
          mbar_wait(&tfull[b], (rc / a.nrb) & 1, 5);
          if (q == 0) PP_ADD(9);
        }
        tc_fence_after();
        const uint32_t racc = lane_base + static_cast<uint32_t>(b * a.npad);
        const bool first = r == 0, last = r == runs - 1;
        // this run's A-row unscale (XW: X row; XTU: X column `row`): power of two
        const float rowf = kHalf ? (a.scan ? rsc[(rc % kRscRing) * kBM + q * 32 + lane] : xinv) : 1.0f;
        {
          // fold the run into L (the last run too: the run buffer is released
          // before the item's output is written from L, so the MMAs of the next
          // item overlap it): 32 columns per TMEM round trip (both loads issued
          // before one wait; the fold is latency-bound otherwise)
          int c0 = c_lo;
          for (; c0 + 32 <= c_hi; c0 += 32) {
            uint32_t rv[32], rs[32];
            tmem_ld32_nowait(racc + c0, rv);
            if (!first) tmem_ld32_nowait(lacc + c0, rs);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              v[e] = __uint_as_float(rv[e]);
              if (kHalf) {  // power-of-two unscale: the FFMA rounds exactly like mul + add
                const float f = kMode == kXTU ? rowf * runsc[c0 + e] : rowf;
                v[e] = first ? v[e] * f : __fmaf_rn(v[e], f, __uint_as_float(rs[e]));
              } else if (!first) {
                v[e] = __fadd_rn(v[e], __uint_as_float(rs[e]));
              }
            }
            tmem_st32(lacc + c0, v);
          }
          if (c0 < c_hi) {
            uint32_t rv[16], rs[16];
            tmem_ld16_nowait(racc + c0, rv);
            if (!first) tmem_ld16_nowait(lacc + c0, rs);
            tmem_ld_wait();
            float v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              v[e] = __uint_as_float(rv[e]);
              if (kHalf) {  // power-of-two unscale: the FFMA rounds exactly like mul + add
                const float f = kMode == kXTU ? rowf * runsc[c0 + e] : rowf;
                v[e] = first ? v[e] * f : __fmaf_rn(v[e], f, __uint_as_float(rs[e]));
              } else if (!first) {
                v[e] = __fadd_rn(v[e], __uint_as_float(rs[e]));
              }
            }
            tmem_st16(lacc + c0, v);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&tempty[b]), 0));
        }
      }
      if (!to_planes16) {
        // the item's output from L: X W rows (row-major fp32, 16 B stores when
        // aligned) or tf32 hi/lo planes of its transpose; X^T U: fp64 partials
        tc_fence_after();
        for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
          float v[16];
          tmem_ld16(lacc + c0, v);
          if (kMode == kXW) {
            if (kHalf) {
#pragma unroll
              for (int e = 0; e < 16; ++e) v[e] *= __ldg(a.winv + c0 + e);
            }
            if (row < a.m) {
              if (a.out_hi) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const float h = tf32_trunc(v[e]);
                  a.out_hi[static_cast<size_t>(c0 + e) * a.ldh + row] = h;
                  a.out_lo[static_cast<size_t>(c0 + e) * a.ldh + row] = tf32_trunc(v[e] - h);
                }
              }
              if (a.out) {
                float* po = a.out + static_cast<size_t>(row) * a.ldo + c0;
                if (c0 + 16 <= a.wstore && (a.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0) {
#pragma unroll
                  for (int e = 0; e < 16; e += 4)
                    *reinterpret_cast<float4*>(po + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                } else {
#pragma unroll
                  for (int e = 0; e < 16; ++e)
                    if (c0 + e < a.wstore) po[e] = v[e];
                }
              }
            }
          } else if (row < a.n) {
            const int ntiles = (a.n + 2 * kBM - 1) / (2 * kBM);
            double* p = a.part + static_cast<size_t>(item / ntiles) * a.l_ld * a.n + static_cast<size_t>(row) * a.l_ld;
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (c0 + e < a.l) p[c0 + e] = static_cast<double>(v[e]);
          }
        }
        tc_fence_before();
      } else {
        // OUT^T as fp16 hi/lo planes scaled per (column, 256-row block = this
        // pair's item): pass 1 reduces each warp's column maxima of the raw
        // accumulator; pass 1.5 combines the four warps, swaps the CTA's
        // maxima with the peer (st.async into the peer's xbuf, completing the
        // peer's xch transaction) and turns the pair maxima into per-column
        // multipliers g[c] = f[c] s[c] (f = the accumulator's own unscale),
        // identical in both CTAs; pass 2 splits.
        tc_fence_after();
        const bool valid = row < a.m;
        float* gsc = red + kMaxEpiWarps * a.npad;
        for (int c0 = c_lo; c0 < c_hi; c0 += 16) {  // rows 0..3 of red: one per lane quadrant
          float v[16];
          tmem_ld16(lacc + c0, v);
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = valid ? fabsf(v[e]) : 0.0f;
          const float mx = warp_max16(v, lane);
          if ((lane & 1) == 0) red[q * a.npad + c0 + warp_max16_col(lane)] = mx;
        }
        epi_bar<kEpiWarps>();
        const int xb = xit & 1;
        if (ew == 0 && lane == 0) mbar_expect_tx(&xch[xb], static_cast<uint32_t>(a.npad) * 4);
        for (int c = ew * 32 + lane; c < a.npad; c += 32 * kEpiWarps) {
          const float mloc = fmaxf(fmaxf(red[c], red[a.npad + c]), fmaxf(red[2 * a.npad + c], red[3 * a.npad + c]));
          gsc[c] = mloc;
          st_async_f32(map_to_rank(smem_u32(&xbuf[xb * a.npad + c]), rank ^ 1u), mloc,
                       map_to_rank(smem_u32(&xch[xb]), rank ^ 1u));
        }
        mbar_wait(&xch[xb], (xit >> 1) & 1, 6);
        ++xit;
        // A scale block is kItemsPerBlock items (kUScaleRows rows), done back to
        // back by this pair (pair_item): the first item's planes go out at its
        // own scale with one bit of headroom; a later item keeps the block's
        // current scale when its maxima fit under it, else settles a smaller
        // one from the block's running maxima and rescales the block's earlier
        // planes (this thread's rows of them) by the ratio, a power of two.
        const int blk = t0 / kUScaleRows;
        const int qi = (t0 / (2 * kBM)) % kItemsPerBlock;  // the item's place in its block
        float* mkeep = red + 4 * a.npad;  // the block's running pair maxima (raw accumulator)
        float* fac = red + 5 * a.npad;    // new scale / previous scale per column
        float* scur = red + 6 * a.npad;   // the block's current scale per column
        // (a pair whose rows all lie past m owns no block: writing its scales
        // would run past the [ceil(m / kUScaleRows)][npad] array)
        for (int c = ew * 32 + lane; c < a.npad; c += 32 * kEpiWarps) {
          const float f = kHalf ? __ldg(a.winv + c) : 1.0f;
          float mraw = fmaxf(gsc[c], xbuf[xb * a.npad + c]);
          float sc;
          if (qi > 0) {
            const float s1 = scur[c];
            if (mraw * f * s1 < 32768.0f) {  // within the block's headroom: its scale stands
              sc = s1;
            } else {
              sc = pow2_scale_for(fmaxf(mraw, mkeep[c]) * f);
            }
            fac[c] = sc / s1;
            mkeep[c] = fmaxf(mkeep[c], mraw);
          } else {
            mkeep[c] = mraw;
            sc = 0.5f * pow2_scale_for(mraw * f);  // one bit of headroom for the block's later items
          }
          scur[c] = sc;
          gsc[c] = f * sc;
          if (rank == 0 && blk * kUScaleRows < a.m) a.uinv[static_cast<size_t>(blk) * a.uinv_ld + c] = __frcp_rn(sc);
        }
        epi_bar<kEpiWarps>();
        for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
          float v[16];
          tmem_ld16(lacc + c0, v);
          if (valid) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int c = c0 + e;
              const float y = v[e] * gsc[c];
              const __half h = __float2half_rn(y);
              a.uh[static_cast<size_t>(c) * a.ldh + row] = h;
              a.ul[static_cast<size_t>(c) * a.ldh + row] = __float2half_rn(y - __half2float(h));
            }
          }
        }
        if (qi > 0) {  // the block's earlier items: this thread's rows of them (written by this thread)
          for (int c = c_lo; c < c_hi; ++c) {
            const float g = fac[c];
            if (g != 1.0f) {
              for (int k = 1; k <= qi; ++k) {
                const size_t r1 = static_cast<size_t>(row - k * 2 * kBM);
                __half* ph = a.uh + static_cast<size_t>(c) * a.ldh + r1;
                __half* pl = a.ul + static_cast<size_t>(c) * a.ldh + r1;
                *ph = __float2half_rn(__half2float(*ph) * g);
                *pl = __float2half_rn(__half2float(*pl) * g);
              }
            }
          }
        }
        tc_fence_before();
        epi_bar<kEpiWarps>();  // red[] reused by the next item
      }
    }
  }
#ifdef LPCA_PAIR_PROF
  {
    const int role = warp == 0 ? 0 : warp == 1 ? 1 : warp == 4 ? 2 : warp == 8 ? 3 : -1;  // q == 0 warps
    if (role >= 0 && lane == 0 && (warp != 1 || leader)) {
      for (int k = 0; k < 16; ++k)
        if (pp[k]) atomicAdd(&g_pair_prof[kMode][k], static_cast<unsigned long long>(pp[k]));
      atomicAdd(&g_pair_prof[kMode][12 + role], static_cast<unsigned long long>(clock64() - pp_start));
    }
  }
#endif
  __syncthreads();
  cluster_sync();  // the peer is done with every barrier and TMEM column
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, a.tmem_cols);
  }
}
