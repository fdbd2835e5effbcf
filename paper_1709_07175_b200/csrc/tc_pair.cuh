// 2-SM (cta_group::2) variant of the split-TF32 pass kernels in gemm_tc.cu.
//
// Why: at the fit's widths (N = 112..224) every 32-deep stage of the 1-SM
// kernel moves the B hi/lo planes (2 * N * 128 B) through L2, TMA and shared
// memory for only 12 MMAs; with M = 128 rows per CTA the B re-reads are
// 1.75x the X bytes and the L2 -> SM traffic saturates (~8 TB/s measured,
// tools/bench_xw.py) well before the MMA floor or HBM. A CTA pair issues
// M = 256 MMAs: each CTA keeps its own 128 rows of A in its TMEM and loads only
// its half of B (N/2 rows); the tensor core reads B from both CTAs' shared
// memory. Per SM, B traffic halves.
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
// Included by gemm_tc.cu inside its anonymous namespace (shares kBM, kBK,
// kRunStages, TcArgs and the tc:: helpers). Pair work items: XW 256-row tiles;
// XTU 256-column tiles x row chunks. Each CTA holds npad / 2 rows of B.
#pragma once

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
// One K=32 stage of the 3-term split as M = 256 pair MMAs (A from TMEM of both CTAs).
__device__ __forceinline__ void mma_stage_ts_pair(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t bh, uint64_t bl,
                                                  uint32_t idesc, uint32_t acc_first) {
#define LPCA_M2 "{%7, %7, %7, %7, %7, %7, %7, %7}"
  asm volatile(
      "{\n .reg .pred p, t;\n setp.ne.b32 p, %6, 0;\n setp.eq.u32 t, %7, %7;\n"
      " .reg .b32 ah, al;\n .reg .b64 dh, dl;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %3, %5, " LPCA_M2 ", p;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%2], %3, %5, " LPCA_M2 ", t;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %4, %5, " LPCA_M2 ", t;\n"
      " add.u32 ah, %1, 8;\n add.u32 al, %2, 8;\n add.u64 dh, %3, 2;\n add.u64 dl, %4, 2;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], dh, %5, " LPCA_M2 ", t;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], dh, %5, " LPCA_M2 ", t;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], dl, %5, " LPCA_M2 ", t;\n"
      " add.u32 ah, %1, 16;\n add.u32 al, %2, 16;\n add.u64 dh, %3, 4;\n add.u64 dl, %4, 4;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], dh, %5, " LPCA_M2 ", t;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], dh, %5, " LPCA_M2 ", t;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], dl, %5, " LPCA_M2 ", t;\n"
      " add.u32 ah, %1, 24;\n add.u32 al, %2, 24;\n add.u64 dh, %3, 6;\n add.u64 dl, %4, 6;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], dh, %5, " LPCA_M2 ", t;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [al], dh, %5, " LPCA_M2 ", t;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [ah], dl, %5, " LPCA_M2 ", t;\n"
      "}" ::"r"(d),
      "r"(a_hi), "r"(a_lo), "l"(bh), "l"(bl), "r"(idesc), "r"(acc_first), "r"(0u)
      : "memory");
#undef LPCA_M2
}

template <int kMode>
__device__ __forceinline__ void pair_item_coords(const TcArgs& a, int item, int& t0, int& k0, int& k1) {
  if (kMode == kXW) {
    t0 = item * 2 * kBM;
    k0 = 0;
    k1 = a.n;
  } else {
    const int ntiles = (a.n + 2 * kBM - 1) / (2 * kBM);
    const int nt = item % ntiles, ch = item / ntiles;
    t0 = nt * 2 * kBM;
    k0 = ch * a.chunk_rows;
    k1 = min(a.m, k0 + a.chunk_rows);
  }
}

template <int kMode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc2_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmbh,
               const __grid_constant__ CUtensorMap tmbl, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages, AS = a.aslots;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  constexpr uint32_t x_bytes = kBM * kBK * 4;                          // this CTA's 128 A rows
  const uint32_t bh_bytes = static_cast<uint32_t>(a.npad / 2) * kBK * 4;  // this CTA's half of B
  const uint32_t stage_bytes = x_bytes + 2 * bh_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* full_x = bars;
  uint64_t* full_b = full_x + S;
  uint64_t* empty = full_b + S;
  uint64_t* conv = empty + S;
  uint64_t* aempty = conv + AS;
  uint64_t* tfull = aempty + AS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t a_col0 = static_cast<uint32_t>((a.nrb + 1) * a.npad);
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

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
      mbar_init(&tempty[b], 8);
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

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int brow = static_cast<int>(rank) * (a.npad / 2);
      for (int item = pair; item < a.items; item += npairs) {
        int t0, k0, k1;
        pair_item_coords<kMode>(a, item, t0, k0, k1);
        const int mine = t0 + static_cast<int>(rank) * kBM;
        for (int k = k0; k < k1; k += kBK) {
          mbar_wait(&empty[stage], phase ^ 1, 1);
          uint8_t* st = smem + stage * stage_bytes;
          mbar_expect_tx(&full_x[stage], x_bytes);
          if (kMode == kXW)
            tma_load_2d(st, &tmx, &full_x[stage], k, mine);
          else
            tma_load_2d(st, &tmx, &full_x[stage], mine, k);
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
      const uint32_t idesc = idesc_tf32(2 * kBM, a.npad, 0, 0);
      const uint64_t desc0 = sw128_desc(smem_u32(smem) + x_bytes, 16, 1024);
      int stage = 0, aslot = 0, rc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int item = pair; item < a.items; item += npairs) {
        int t0, k0, k1;
        pair_item_coords<kMode>(a, item, t0, k0, k1);
        for (int q0 = k0; q0 < k1; q0 += kRunStages * kBK, ++rc) {
          const int b = rc % a.nrb;
          mbar_wait(&tempty[b], ((rc / a.nrb) & 1) ^ 1, 2);
          tc_fence_after();
          const uint32_t d = tmem_base + static_cast<uint32_t>(b * a.npad);
          const int q1 = min(k1, q0 + kRunStages * kBK);
          for (int k = q0; k < q1; k += kBK) {
            mbar_wait(&conv[aslot], aphase, 3);
            mbar_wait(&full_b[stage], phase, 3);
            tc_fence_after();
            const uint64_t bh = desc0 + static_cast<uint64_t>((stage * stage_bytes) >> 4);
            const uint64_t bl = bh + static_cast<uint64_t>(bh_bytes >> 4);
            const uint32_t at = tmem_base + a_col0 + static_cast<uint32_t>(aslot * 64);
            if (elect_one()) {
              mma_stage_ts_pair(d, at, at + 32, bh, bl, idesc, k != q0 ? 1u : 0u);
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
  } else if (warp < 6) {
    // ---------------- converters (both CTAs): smem X -> own TMEM A ----------------
    const int q = warp & 3;
    const int i = q * 32 + lane;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    int stage = 0, aslot = 0;
    uint32_t phase = 0, aphase = 0;
    for (int item = pair; item < a.items; item += npairs) {
      int t0, k0, k1;
      pair_item_coords<kMode>(a, item, t0, k0, k1);
      for (int k = k0; k < k1; k += kBK) {
        mbar_wait(&full_x[stage], phase, 4);
        mbar_wait(&aempty[aslot], aphase ^ 1, 4);
        tc_fence_after();
        const uint8_t* xt = smem + stage * stage_bytes;
        float v[32];
        if (kMode == kXW) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 f = *reinterpret_cast<const float4*>(xt + i * 128 + ((c ^ (i & 7)) << 4));
            v[4 * c] = f.x;
            v[4 * c + 1] = f.y;
            v[4 * c + 2] = f.z;
            v[4 * c + 3] = f.w;
          }
        } else {
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
        if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&conv[aslot]), 0));
        ring_advance(stage, phase, S);
        ring_advance(aslot, aphase, AS);
      }
    }
  } else {
    // ---------------- epilogue (both CTAs, own 128 rows) ----------------
    const int q = warp & 3;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t lacc = lane_base + static_cast<uint32_t>(a.nrb * a.npad);
    int rc = 0;
    for (int item = pair; item < a.items; item += npairs) {
      int t0, k0, k1;
      pair_item_coords<kMode>(a, item, t0, k0, k1);
      const int runs = (k1 - k0 + kRunStages * kBK - 1) / (kRunStages * kBK);
      const int row = t0 + static_cast<int>(rank) * kBM + q * 32 + lane;
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
            const int ntiles = (a.n + 2 * kBM - 1) / (2 * kBM);
            double* p = a.part + static_cast<size_t>(item / ntiles) * a.l * a.n + static_cast<size_t>(row) * a.l;
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (c0 + e < a.l) p[c0 + e] = static_cast<double>(v[e]);
          }
        }
        if (!last) tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(map_to_rank(smem_u32(&tempty[b]), 0));
      }
    }
  }
  __syncthreads();
  cluster_sync();  // the peer is done with every barrier and TMEM column
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, a.tmem_cols);
  }
}

