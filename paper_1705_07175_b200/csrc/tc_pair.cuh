// CTA-pair (cta_group::2) binary GEMM on the fp4 tensor cores.
//
// The single-CTA kernel (k_tc_gemm, 128 x 256 tiles) moves ~192 bytes of
// shared memory per clock at the full kind::mxf4 rate — the MMA reads A and B
// (96 B/clk), the producer warps write the expanded A (32 B/clk) and TMA
// writes B (64 B/clk) — while an SM's shared memory delivers 128 B/clk, so
// the tensor pipe cannot run above ~2/3 of its rate (ncu: 57 % busy on BCNN
// conv4 / conv6).  Two CTAs on the two SMs of a TPC share one 256 x 256 tile:
// `tcgen05.mma.cta_group::2` (M = 256) reads A rows 0-127 from CTA 0's shared
// memory and rows 128-255 from CTA 1's, and B columns 0-127 from CTA 0 and
// 128-255 from CTA 1, and each CTA's tensor memory holds the accumulator of
// its own 128 rows.  Per SM and stage that is 32 KB read by the MMA + 16 KB of
// expanded A + 16 KB of B = 128 B/clk at the full rate: a third less traffic
// for the same MACs.
//
// Roles (both CTAs, 640 threads): warp 0 lane 0 = TMA of this CTA's B half;
// warp 1 lane 0 = MMA issuer (CTA 0) / "stage ready" relay (CTA 1: waits for
// its own stage to fill and arrives on CTA 0's barrier); warp 2 = TMEM
// allocator (cta_group::2); warps 4-11 = A producers of this CTA's 128 rows
// (the single-CTA producer code, ACursor); warps 12-19 = epilogue of this
// CTA's rows.  MMA completion is committed to both CTAs' barriers at once
// (multicast); the epilogues of both CTAs release the accumulator on CTA 0's
// barrier.
#pragma once
#include "tc_i8.cuh"

namespace b2 {
namespace tc {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Arrive on the peer CTA's mbarrier.  Relaxed: a .release.cluster arrive
// compiles to a GPU-scope MEMBAR + ERRBAR (measured: the dominant stall of the
// relay thread), and the waits pair with plain (CTA-scope) try_waits — an
// .acquire.cluster wait invalidates the SM's whole L1 (CCTL.IVALL) every time,
// flushing the producers' cached input rows.  What the arrive publishes is
// already ordered: the stage data by the producers' fence.proxy.async and
// their release arrive on the local barrier the relay acquired, the
// accumulator reads by tcgen05.wait::ld + tcgen05.fence::before_thread_sync.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tc_mma_f4_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t sfa_tmem, uint32_t sfb_tmem, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // arrive on `bar` in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// instruction descriptor, kind::mxf4 with M = 256 (cta_group::2)
__host__ __device__ constexpr uint32_t idesc_f4_pair(int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((256u >> 4) << 24);
}

constexpr int PAIR_BN = 256, PAIR_BKS = 256, PAIR_NPW = 8, PAIR_NEPI = 8;
constexpr int PAIR_A_BYTES = BM * PAIR_BKS / 2;        // 16 KB: this CTA's 128 A rows of one K stage
constexpr int PAIR_B_BYTES = (PAIR_BN / 2) * PAIR_BKS / 2;  // 16 KB: this CTA's 128 B rows
constexpr int PAIR_STAGES = (192 * 1024) / (PAIR_A_BYTES + PAIR_B_BYTES);  // 6
constexpr int pair_smem_bytes() {
  return PAIR_STAGES * (PAIR_A_BYTES + PAIR_B_BYTES) + THR_COLS * 8 + THR_COLS / 8 + 8 * (3 * PAIR_STAGES + 4) + 16 +
         1024;
}

template <int AM, int EM>
__global__ void __launch_bounds__(32 * (4 + PAIR_NPW + PAIR_NEPI), 1)
    k_pair_gemm(const __grid_constant__ CUtensorMap bmap, const Args g) {
  constexpr int BN = PAIR_BN, BKS = PAIR_BKS, NPW = PAIR_NPW, NEPI = PAIR_NEPI;
  constexpr int WS = BKS / 32;       // K words per stage
  constexpr int HALVES = NPW / 4;    // producer warps per lane quarter
  constexpr int WPH = WS / HALVES;   // K words per producer thread per stage
  constexpr int EPI0 = 4 + NPW;
  constexpr bool POOLED = (EM == E_POOLPACK);
  constexpr int SA = PAIR_STAGES;
  constexpr int SF_COL = BN;  // one accumulator, unit scale factors after it
  constexpr uint32_t IDESC = idesc_f4_pair(BN);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sb = smem;                                  // SA x PAIR_B_BYTES (this CTA's B half)
  uint8_t* sa = smem + SA * PAIR_B_BYTES;              // SA x PAIR_A_BYTES (this CTA's A rows)
  int4* sthr = reinterpret_cast<int4*>(sa + SA * PAIR_A_BYTES);
  uint32_t* sgm = reinterpret_cast<uint32_t*>(sthr + THR_COLS / 2);
  uint64_t* full = reinterpret_cast<uint64_t*>(sgm + THR_COLS / 32);
  uint64_t* pfull = full + SA;   // CTA 0: the peer's stage s is full (relay)
  uint64_t* empty = pfull + SA;
  uint64_t* tfull = empty + SA;
  uint64_t* tempty = tfull + 1;  // CTA 0: both CTAs' epilogues released the accumulator
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t mtiles = (g.M + 2 * BM - 1) / (2 * BM);  // 256-row tiles
  const int ntiles = (g.N + BN - 1) / BN;
  const int64_t tiles = mtiles * ntiles;  // tile T -> (m tile T % mtiles, n tile T / mtiles)
  // this CTA's 128-row half of tile T is "tile" 2 T + rank of a 128-row tiling
  // with 2 mtiles m tiles (ACursor's view; the last half may lie past M)
  const int64_t mtiles2 = 2 * mtiles, tiles2 = 2 * tiles;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&full[s], NPW + 1);  // producer warps + the TMA expect_tx arrival
      mbar_init(&pfull[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * NEPI);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&bmap) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {  // unit block scales (e8m0 0x7F) in this CTA's lanes
    uint32_t ones[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) ones[i] = 0x7F7F7F7Fu;
    tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + SF_COL, ones);
    tmem_wait_st();
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers and scale factors exist before any remote access
  tc_fence_after();
  pdl_entry();
  // registers by role (per warpgroup): the control warps and the producers
  // give theirs to the epilogue, which holds all 128 accumulator columns of
  // its rows at once so the accumulator returns to the MMA after one TMEM
  // round trip (it is single-buffered: 256 columns + scale factors)
  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");

  if (warp == 0) {
    // ------------------------------------------------ TMA: this CTA's half of B
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      // L2 prefetch of the A inputs this CTA's producers gather, two tiles ahead
      prefetch_tile_inputs<AM>(g, 2 * pair + rank, mtiles2, tiles2);
      prefetch_tile_inputs<AM>(g, 2 * (pair + npairs) + rank, mtiles2, tiles2);
      for (int64_t t = pair; t < tiles; t += npairs) {
        prefetch_tile_inputs<AM>(g, 2 * (t + 2 * npairs) + rank, mtiles2, tiles2);
        const int n0 = (int)(t / mtiles) * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < g.nkb; ++kb) {
          mbar_wait_nc(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], PAIR_B_BYTES);
          tma_load_2d(sb + s * PAIR_B_BYTES, &bmap, &full[s], kb * BKS / 2, n0);
          if (++s == SA) s = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      if (rank == 0) {
        // ---------------------------------------------- MMA issuer (CTA 0)
        uint32_t aph = 0;
        for (int64_t t = pair; t < tiles; t += npairs) {
          mbar_wait(tempty, aph ^ 1);
          tc_fence_after();
          for (int kb = 0; kb < g.nkb; ++kb) {
            mbar_wait(&full[s], ph);
            mbar_wait(&pfull[s], ph);
            tc_fence_after();
            const uint32_t as = smem_u32(sa + s * PAIR_A_BYTES), bs = smem_u32(sb + s * PAIR_B_BYTES);
            const int kmma = kb + 1 == g.nkb ? g.klast : BKS / 64;
#pragma unroll
            for (int k = 0; k < BKS / 64; ++k)
              if (k < kmma)
                tc_mma_f4_pair(tmem, sw128_desc(as + (k >> 2) * BM * BK + (k & 3) * 32),
                               sw128_desc(bs + (k >> 2) * (BN / 2) * BK + (k & 3) * 32), IDESC, tmem + SF_COL,
                               tmem + SF_COL + 4, (kb > 0 || k) ? 1u : 0u);
            tc_commit_pair(&empty[s]);
            if (++s == SA) s = 0, ph ^= 1;
          }
          tc_commit_pair(tfull);
          aph ^= 1;
        }
      } else {
        // ---------------------------------------------- relay (CTA 1): my stage s is full
        const uint32_t peer_pfull = cluster_map(smem_u32(pfull), 0);
        for (int64_t t = pair; t < tiles; t += npairs)
          for (int kb = 0; kb < g.nkb; ++kb) {
            mbar_wait(&full[s], ph);
            mbar_arrive_remote(peer_pfull + 8u * (uint32_t)s);
            if (++s == SA) s = 0, ph ^= 1;
          }
      }
    }
  } else if (warp >= 4 && warp < EPI0) {
    // ------------------------------------------------ A producers (this CTA's 128 rows)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    ACursor<AM, POOLED, WS, WPH, AM == A_CONV> cur;
    const int64_t step2 = 2 * npairs;
    cur.start(g, 2 * pair + rank, mtiles2, tiles2, r, half, 1);
    const int64_t my_tiles = pair < tiles ? (tiles - 1 - pair) / npairs + 1 : 0;
    const int jobs = (int)(my_tiles * g.nkb);
    constexpr int PFQ = 4;
    uint4 qx[PFQ];
    bool qok[PFQ];
#pragma unroll
    for (int u = 0; u < PFQ; ++u) {
      uint4 vm;
      cur.template fetch_bits<WPH>(g, half, qx[u], vm);
      qok[u] = vm.x != 0 || vm.y != 0 || vm.z != 0 || vm.w != 0;
      cur.advance(g, step2, mtiles2, tiles2, r, half, 1);
    }
    int s = 0;
    uint32_t ph = 0;
    for (int j0 = 0; j0 < jobs; j0 += PFQ) {
#pragma unroll
      for (int u = 0; u < PFQ; ++u) {
        if (j0 + u < jobs) {
          uint32_t v[4 * WPH];
          widen_f4(qx[u].x, qok[u], v + 0);
          widen_f4(qx[u].y, qok[u], v + 4);
          if constexpr (WPH == 4) {
            widen_f4(qx[u].z, qok[u], v + 8);
            widen_f4(qx[u].w, qok[u], v + 12);
          }
          uint4 vm;
          cur.template fetch_bits<WPH>(g, half, qx[u], vm);
          qok[u] = vm.x != 0 || vm.y != 0 || vm.z != 0 || vm.w != 0;
          cur.advance(g, step2, mtiles2, tiles2, r, half, 1);
          mbar_wait_nc(&empty[s], ph ^ 1);
          uint8_t* row = sa + s * PAIR_A_BYTES + r * 128;
          const int wend = g.nkb == 1 ? 2 * g.klast : WS;
#pragma unroll
          for (int i = 0; i < WPH; ++i) {
            const int w = half * WPH + i;
            if (w < wend)
              *reinterpret_cast<uint4*>(row + (w >> 3) * (BM * 128) + (((w & 7) ^ (r & 7)) << 4)) =
                  make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
          if (++s == SA) s = 0, ph ^= 1;
        }
      }
    }
  } else if (warp >= EPI0) {
    // ------------------------------------------------ epilogue (this CTA's 128 rows)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 160;");
    constexpr int ECOLS = BN / (NEPI / 4);  // 128 columns per warp
    constexpr int ECH = ECOLS / 32;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int ec0 = ((warp - EPI0) >> 2) * ECOLS;
    const int et = (warp - EPI0) * 32 + lane;
    const uint32_t lane_addr = ((uint32_t)(q * 32) << 16) + ec0;
    const uint32_t peer_tempty = cluster_map(smem_u32(tempty), 0);
    auto release = [&]() {  // this warp is done reading the accumulator
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(tempty);
        else
          mbar_arrive_remote(peer_tempty);
      }
    };
    uint32_t aph = 0;
    const int ncols = ntiles * BN;
    const bool static_thr = ncols <= THR_COLS;
    if constexpr (EM == E_PACK || EM == E_POOLPACK) {
      if (static_thr) {
        stage_thresholds<true>(g, 0, ncols, et, 32 * NEPI, lane, sthr, sgm);
        epi_bar<NEPI>();
      }
    }
    for (int64_t t = pair; t < tiles; t += npairs) {
      const int64_t mt = 2 * (t % mtiles) + rank;  // this CTA's 128-row block
      const int64_t m = mt * BM + r;
      const int n0 = (int)(t / mtiles) * BN;
      const int tcol = static_thr ? n0 : 0;
      const bool mok = m < g.M;
      if constexpr (EM == E_PACK || EM == E_POOLPACK) {
        if (!static_thr) {
          epi_bar<NEPI>();
          stage_thresholds<true>(g, n0, BN, et, 32 * NEPI, lane, sthr, sgm);
          epi_bar<NEPI>();
        }
      }
      // one warp polls the accumulator barrier, the others block on the
      // epilogue's named barrier (eight polling warps were ~16 % of the
      // kernel's issued instructions)
      if (warp == EPI0) mbar_wait(tfull, aph);
      epi_bar<NEPI>();
      tc_fence_after();
      uint32_t words[ECH];
      const int4* trow = sthr + ((tcol + ec0) >> 1);
      // all chunks at once (one TMEM round trip before the release), except
      // the float64 epilogue, whose per-chunk doubles need the registers:
      // chunk c + 1 in flight while chunk c is processed
      constexpr bool ALL = (EM == E_PACK || EM == E_POOLPACK);
      uint32_t vall[ALL ? ECH : 2][32];
      if constexpr (ALL) {
#pragma unroll
        for (int c = 0; c < ECH; ++c) tmem_ld32(tmem + lane_addr + c * 32, vall[c]);
        tmem_wait_ld();
        release();
      } else {
        tmem_ld32(tmem + lane_addr, vall[0]);
        tmem_wait_ld();
      }
#pragma unroll
      for (int c = 0; c < ECH; ++c) {
        uint32_t(&v)[32] = vall[ALL ? c : (c & 1)];
        if constexpr (!ALL) {
          if (c + 1 < ECH) tmem_ld32(tmem + lane_addr + (c + 1) * 32, vall[(c + 1) & 1]);
        }
        const int nb = n0 + ec0 + c * 32;
        if constexpr (EM == E_AFFINE) {
          if (mok && nb < g.N) {
            double* o = g.out_f64 + m * g.ldo + nb;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = nb + j;
              if (n < g.N)
                o[j] = __dadd_rn(__dmul_rn(__dsub_rn((double)acc_int<true>(v[j]), __ldg(g.mean + n)), __ldg(g.scale + n)),
                                 __ldg(g.beta + n));
            }
          }
        } else if constexpr (EM == E_I32) {
          if (mok && nb < g.N) {
            int32_t* o = g.out_i32 + m * g.ldo + nb;
            if (nb + 32 <= g.N && ((g.ldo & 3) == 0)) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<int4*>(o + j) = make_int4(acc_int<true>(v[j]), acc_int<true>(v[j + 1]),
                                                            acc_int<true>(v[j + 2]), acc_int<true>(v[j + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < g.N) o[j] = acc_int<true>(v[j]);
            }
          }
        } else {
          uint32_t w = thr_word<true>(v, trow + c * 16);
          if constexpr (EM == E_POOLPACK) w = pool_word(w, sgm[((tcol + ec0) >> 5) + c]);
          words[c] = w;
        }
        if constexpr (!ALL) {
          if (c + 1 < ECH) tmem_wait_ld();
          if (c + 2 == ECH) release();
        }
      }
      if constexpr (EM == E_PACK || EM == E_POOLPACK) {
        const int64_t site = POOLED ? (m >> 2) : m;
        if (mok && (!POOLED || (lane & 3) == 0)) {
          const int w0 = (n0 + ec0) / 32;
          uint32_t* o = g.out_bits + site * g.ldo32 + w0;
          if (w0 + ECH <= g.ldo32 && (g.ldo32 & 3) == 0) {
#pragma unroll
            for (int c = 0; c < ECH; c += 4)
              *reinterpret_cast<uint4*>(o + c) = make_uint4(words[c], words[c + 1], words[c + 2], words[c + 3]);
          } else {
#pragma unroll
            for (int c = 0; c < ECH; ++c)
              if (w0 + c < g.ldo32) o[c] = words[c];
          }
        }
      }
      aph ^= 1;
    }
  }
  // no CTA may leave while its peer can still touch its shared or tensor memory
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tc
}  // namespace b2
