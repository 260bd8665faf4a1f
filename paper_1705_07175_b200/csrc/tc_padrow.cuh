// Padded-row implicit GEMM for stride-1 "same" convolutions on the fp4
// tensor cores (tcgen05.mma kind::mxf4).
//
// The im2col producers of k_tc_gemm expand every input word once per window
// cell (9x for 3x3).  Here the output pixels are laid out on a VIRTUAL grid
// whose rows are W + 1 wide (one shared zero column) and whose images are
// H + 1 rows tall (one shared zero row): v(n, y, x) = n (H+1)(W+1) + y (W+1)
// + x.  The input of window cell (dy, dx) for output v is then v + dy (W+1)
// + dx for EVERY v, so one expanded copy of the input band (the virtual rows
// a 128-row tile touches, ±(W+2)) serves all cells: cell (dy, dx) is an MMA
// descriptor whose start is shifted by that many rows.  The band uses the
// no-swizzle K-major canonical layout (8-row x 16-byte core matrices, rows
// 16 bytes apart, one 16-byte K plane per input word), in which a shift by
// any number of rows is a plain start-address offset.
//
// Virtual rows at the zero column / zero row produce accumulators that are
// discarded (W=32: 9.6 % of the MMA work).  A 2x2 pool window spans rows v
// and v + W + 1, which may sit in different tiles, so pooled layers write
// the thresholded bits unpooled and k_pool_bits combines each window (OR for
// ge channels, AND for le: exact, the threshold is monotone).
//
// Scope: fp4, c % 128 == 0, N <= 128 (one 128-column tile), weights
// resident in shared memory (K <= 1536), odd square-or-not windows with
// pad = (k - 1) / 2, stride 1.
#pragma once
#include <cstdio>

#include "tc_pair.cuh"

namespace b2 {
namespace tc {

struct PadArgs {
  const uint32_t* x;   // NHWC-bits input, sstride words per pixel
  int N, H, W, sstride, P;  // P = c / 32 words (= K planes) per pixel
  int kh, kw, pad;
  int Wp;              // W + pad (pad zero columns per virtual row)
  int64_t VI, Vtotal;  // virtual rows per image, in all
  uint64_t vi_magic;   // ceil(2^64 / VI): image of a virtual row by one multiply-high
  uint32_t wp_magic;   // ceil(2^32 / Wp): row within the image
  int R8;              // band rows (multiple of 8): 128 + 2 * band0
  int band0;           // halo above a tile: pad * Wp + pad virtual rows
  int nkb;             // 128-byte B atoms (256 K elements) in shared memory
  int nkb_ld;          // ALIGN: atoms loaded from the weights (nkb may add one for the threshold block); 0 = nkb
  int kk;              // ALIGN: K = kh kw c (the threshold block's first K element)
  int band_bytes;      // band slot stride: max(PR_BAND_MAX, R8 * 16 * planes) rounded to 1 KB
  int F;               // filters (<= 128)
  int kmmas;           // K=64 MMAs per window cell (= P / 2)
  uint32_t* out_bits;  // (N*H*W, ldo32) words
  int64_t ldo32;
  const int32_t* thresh;
  const uint8_t* ge;
  // BYTEIN (byte-BN first layer): u8 image (N, H, W, cin), per-channel
  // byte thresholds; one data plane per pixel (cin <= 8 bits) + a zero plane
  const uint8_t* xb;
  int cin;
  const int32_t* th_in;
  const uint8_t* ge_in;
  // ALIGN (row-aligned tiles): a tile is 128 consecutive pixels of one image
  // (128 / W whole rows, W | 128, 128 | H W); the band holds kw copies of the
  // tile's input rows (+-pad rows), copy dx shifted by dx - pad columns with
  // zeros past the row ends, so window cell (dy, dx) is copy dx at a shift
  // of dy W rows: no virtual zero column / row, and a 2x2 pool window lies
  // inside one tile (fused into the epilogue)
  int64_t HW;          // pixels per image
  int wshift;          // log2 W
  int Rb;              // band rows per copy: (128 / W + 2 pad) W
  int nbands;          // band slots in the ring (<= PR_BANDS_MAX)
  int pool;            // fused 2x2/2 max-pool (OR ge / AND le of thresholded bits)
  int pair;            // CTA-pair launch (PAIR kernel), set by the host plan
  int raw;             // ALIGN: input rows through the loader warp's staging ring (0: register prefetch)
  int wlim;            // output words this launch writes per pixel (0: ldo32; a filter split's part writes its own)
  // TW (row-aligned, filters on the MMA's M side): the weights live in TMEM,
  // read once from these fp4 rows (wt_words 32-bit words = K / 8 of each
  // row, rows wt_stride words apart)
  int tw;
  const uint32_t* wt;
  int wt_words;
  int wt_stride;
};

#ifndef B2_PADROW_LBO_K
#define B2_PADROW_LBO_K 1  // 1: LBO = K-plane stride, SBO = 8-row group stride (0: swapped)
#endif

// K-major, no swizzle: 8-row x 16-byte core matrices
__device__ __forceinline__ uint64_t noswz_desc(uint32_t saddr, uint32_t kplane_bytes) {
  const uint64_t lbo = B2_PADROW_LBO_K ? kplane_bytes : 128u, sbo = B2_PADROW_LBO_K ? 128u : kplane_bytes;
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// virtual row v -> (image n, row y, column x) of the padded grid
__device__ __forceinline__ void vsplit(const PadArgs& g, int64_t v, int64_t& n, int& y, int& x) {
  n = (int64_t)__umul64hi((uint64_t)v, g.vi_magic);
  const uint32_t rem = (uint32_t)(v - n * g.VI);
  y = (int)__umulhi(rem, g.wp_magic);
  x = (int)rem - y * g.Wp;
}

constexpr int PR_NPW = 8;       // producer warps
#ifndef B2_PR_PROD_POLL  // ALIGN producers' band-empty wait: 0 back off (nanosleep), 1 poll, 2 suspend hint
#define B2_PR_PROD_POLL 0
#endif
#ifndef B2_PR_SLEEP_NS  // back-off of the ALIGN loader / producer waits (ncu: the suspend-hinted try_wait
#define B2_PR_SLEEP_NS 128  // still retried ~25 times per tile per warp, ~11 % of the kernel's issued instructions)
#endif
#if B2_PR_PROD_POLL == 1
#define B2_PR_PROD_WAIT(b, p) mbar_wait(b, p)
#elif B2_PR_PROD_POLL == 2
#define B2_PR_PROD_WAIT(b, p) mbar_wait_suspend(b, p)
#else
#define B2_PR_PROD_WAIT(b, p) mbar_wait_sleep(b, p, B2_PR_SLEEP_NS)
#endif
#ifndef B2_PR_EPI_SUSPEND  // epilogue waits: 1 suspend in hardware, 0 poll
#define B2_PR_EPI_SUSPEND 0
#endif
#ifndef B2_PR_NEPI
#define B2_PR_NEPI 4
#endif
#ifndef B2_PR_NEPI_ALIGN  // epilogue warps of the 128-column row-aligned kernel
#define B2_PR_NEPI_ALIGN 4  // 4: conv2 / conv3 ~1 % faster than 8
#endif
#ifndef B2_PR_DRAIN2  // bias-folded 256-column padded-row kernels: two-round-trip drain
#define B2_PR_DRAIN2 0  // measured no faster on conv3 (1.62 vs 1.61 ms)
#endif
#ifndef B2_PR_VBIAS  // virtual-grid kernel: threshold folded into the GEMM too
#define B2_PR_VBIAS 0  // measured slower on conv3 (1.80 vs 1.66 ms): one more 128-cycle MMA per tile for an epilogue that was not the limit
#endif
#ifndef B2_PR_WI_ALL  // virtual-grid kernel: warp-wide MMA issue too
#define B2_PR_WI_ALL 0
#endif
#ifndef B2_PR_WARP_ISSUE
#define B2_PR_WARP_ISSUE 1
#endif
constexpr int PR_NEPI = B2_PR_NEPI;  // epilogue warps: 4 (one per lane quarter) or 8 (two, half the columns each)
constexpr int PR_BANDS = 4;     // band ring (tiles in flight: hides the band loads' DRAM latency)
constexpr int PR_ACC = 3;       // accumulator buffers (3 x 128 columns + scale columns)
constexpr int PR_BAND_MAX = 16 * 1024;  // bytes per band slot (the minimum; wider images take larger slots)
constexpr int PR_BANDS_MAX = 4;         // barrier slots reserved for the band ring
#ifndef B2_PR_RAW_SLOTS
#define B2_PR_RAW_SLOTS 4
#endif
constexpr int PR_RAW_SLOTS = B2_PR_RAW_SLOTS;  // ALIGN: raw input staging slots (bulk copies up to this many tiles ahead)

// 1-D bulk copy global -> shared, completion (bytes) on `bar` (16-byte
// aligned addresses and size)
__device__ __forceinline__ void bulk_g2s_pr(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// KH, KMMAS > 0: compile-time window and K chunks per cell (the issuing
// thread's 18 descriptor offsets for 3x3 / c = 128 stay in registers and the
// MMA loop is fully unrolled: a runtime loop reading them from shared memory
// issued one MMA per ~113 cycles, slower than the 64-cycle MMA itself)
// BNT = 128: three 128-column accumulators, PR_NEPI epilogue warps, four
// band slots; BNT = 256 (up to 256 filters, weights <= 160 KB): one
// 256-column accumulator (2 x 256 + the scale columns exceed TMEM), eight
// epilogue warps, three band slots.
template <int BNT, bool ALIGN = false, bool TW = false>
constexpr int pr_nepi() {  // row-aligned 128-column tiles: B2_PR_NEPI_ALIGN warps (TW: two per lane quarter)
  return BNT == 256 ? 8 : (TW ? 8 : (ALIGN ? B2_PR_NEPI_ALIGN : PR_NEPI));
}
template <int BNT>
constexpr int pr_acc() {
  return BNT == 256 ? 1 : PR_ACC;
}
template <int BNT>
constexpr int pr_bands() {
  return BNT == 256 ? 3 : PR_BANDS;
}

// PAIR (row-aligned only): a CTA pair on the two SMs of a TPC runs each MMA
// as M = 256 (cta_group::2): CTA r computes the 128-pixel tile 2 T + r of pair
// tile T from its own band, and holds half the filters' weights (N / 2 rows),
// so per SM the MMA reads half the weight bytes and the freed shared memory
// buys a deeper band ring (MMA-thread timing of the single-CTA conv2: 23 % of
// its time waiting for a band with three slots).  CTA 1's "band ready" reaches
// CTA 0's issuer through a relay thread (relaxed remote arrive, see
// tc_pair.cuh), MMA completion is committed to both CTAs, and both epilogues
// release the accumulators on CTA 0's barriers.
// Threshold folded into the GEMM (row-aligned single-CTA kernels): one more
// K = 64 MMA per tile adds a per-filter integer bias -T' to every
// accumulator, so the epilogue only collects sign bits (ncu: the kernel was
// issue-bound and the (mul, add) threshold pass was a third of the
// epilogue's instructions).  A = a constant +1 block, B = the filter's 64
// bias elements: block 0 (scale 2^5) holds 16 q, block 1 (scale 2^0) the rest
// r, with b = 16 q + r.  T' = T (ge: bit = acc >= T, i.e. sign clear) or
// T + 1 (le: bit = acc <= T, i.e. sign set), clamped to +-(K + 1).
// TW (row-aligned, BNT = 128, single CTA): the GEMM transposed — D[filter][pixel]
// = W[filter][k] X[pixel][k] with the weights as the A operand in TMEM (loaded
// once, columns PR_TW_COL..) and the band as the B operand.  The MMA then reads
// only the band from shared memory (64 B/clk instead of 128 at N = 128:
// ncu put the tensor pipe's shared-memory wavefronts plus the producers' and
// the threshold reads at ~94 % of the shared-memory pipe), the thresholds are
// per lane (one filter per TMEM lane) and the epilogue transposes sign bits
// with warp ballots, pooling by shuffles with no shared-memory exchange.
constexpr int PR_TW_COL = 288;  // first TMEM column of the resident weights (K / 8 columns, <= 224)
__device__ __forceinline__ void tc_mma_f4_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t sfa_tmem, uint32_t sfb_tmem, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem)
      : "memory");
}

template <int KH, int KMMAS, int BNT, bool BYTEIN = false, bool ALIGN = false, bool PAIR = false, bool TW = false>
__global__ void __launch_bounds__(32 * (4 + PR_NPW + pr_nepi<BNT, ALIGN, TW>()), 1)
    k_padrow_conv(const __grid_constant__ CUtensorMap bmap, const PadArgs g) {
  constexpr int BN = BNT;
  constexpr int BNH = PAIR ? BN / 2 : BN;  // weight rows held by this CTA
  constexpr int PR_NEPI = pr_nepi<BNT, ALIGN, TW>();
  constexpr int PR_ACC = TW ? 2 : pr_acc<BNT>();  // TW: 2 x 128 accumulator columns, scales, then the weights
  static_assert(!(ALIGN && BYTEIN), "row-aligned tiles take packed-bit input");
  static_assert(!PAIR || ALIGN, "CTA pairs only on row-aligned tiles");
  static_assert(!TW || (ALIGN && !PAIR && BNT == 128), "TMEM weights: row-aligned single-CTA 128-pixel tiles");
  constexpr bool BIAS = !PAIR && !TW && !BYTEIN && (ALIGN || B2_PR_VBIAS);  // threshold folded into the GEMM
  const int PR_BANDS = ALIGN ? g.nbands : pr_bands<BNT>();
  constexpr uint32_t IDESC = PAIR ? idesc_f4_pair(BN) : idesc_f4(BN);
  constexpr int EPI0 = 4 + PR_NPW;
  constexpr int ACC_COLS = BN;
  constexpr int SF_COL = PR_ACC * ACC_COLS;
  constexpr int SF_BIAS = SF_COL + 16;  // BIAS: the threshold block's B scales (16 columns)
  static_assert(!BIAS || SF_BIAS + 16 <= (BNT == 256 ? 288 : 512), "TMEM: scale columns");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sb = smem;                                    // resident weights: nkb atoms of BNH x 128 B
  uint8_t* sband = sb + (TW ? 0 : g.nkb * BNH * 128);    // PR_BANDS x band_bytes
  int4* sthr = reinterpret_cast<int4*>(sband + PR_BANDS * g.band_bytes);  // 64 x (mul, add) pairs
  uint32_t* sgm = reinterpret_cast<uint32_t*>(sthr + BN / 2);
  uint64_t* bres = reinterpret_cast<uint64_t*>(sgm + BN / 32);
  uint64_t* bfull = bres + 1;
  uint64_t* bempty = bfull + PR_BANDS_MAX;
  uint64_t* tfull = bempty + PR_BANDS_MAX;
  uint64_t* tempty = tfull + PR_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + PR_ACC);
  uint2* soff = reinterpret_cast<uint2*>(tmem_slot + 2);  // per MMA: (A, B) descriptor address offsets (16 B units)
  uint64_t* bbias = reinterpret_cast<uint64_t*>(soff + 128);  // BIAS: threshold block written
  uint8_t* sones = reinterpret_cast<uint8_t*>(bbias + 2);      // BIAS: 128 rows x 64 e2m1 +1 (4 KB, no swizzle)
  sones += (128u - (smem_u32(sones) & 127u)) & 127u;
  const bool bias_on = BIAS && g.kk > 0;  // the plan may leave the threshold in the epilogue (shared memory)
  uint2* spool = reinterpret_cast<uint2*>(sones + (bias_on ? 4096 : 0));  // ALIGN + pool: [2 tiles][128 rows][BN / 32] (OR, AND)
  uint64_t* pbfull = reinterpret_cast<uint64_t*>(spool + (g.pool || PAIR ? 2 * BM * (BN / 32) : 0));  // PAIR, CTA 0: the peer's band is full
  uint64_t* rfull = pbfull + PR_BANDS_MAX;                                       // ALIGN: raw input staging slot landed
  uint64_t* rempty = rfull + PR_RAW_SLOTS;                                       // ALIGN: every producer warp read it
  uint8_t* sraw = reinterpret_cast<uint8_t*>(rempty + PR_RAW_SLOTS);
  sraw += (16u - (smem_u32(sraw) & 15u)) & 15u;
  // ^ ALIGN: PR_RAW_SLOTS x Rb pixels (16-byte aligned bulk-copy targets)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = ALIGN ? (int64_t)g.N * g.HW / BM : (g.Vtotal + BM - 1) / BM;
  const uint32_t plane_bytes = (uint32_t)g.R8 * 16u;
  // this CTA's tiles: t = t_first, t_first + t_step, ... while the pair tile
  // exists (t - rank < tiles); a PAIR half past the end (odd tile count) is
  // computed on a zero band and not stored
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const int64_t t_first = PAIR ? 2 * (int64_t)(blockIdx.x >> 1) + rank : (int64_t)blockIdx.x;
  const int64_t t_step = PAIR ? 2 * (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;

  if (warp == 0 && lane == 0) {
    mbar_init(bres, TW ? PR_NEPI : 1);  // TW: every epilogue warp has stored its weight rows
    for (int b = 0; b < PR_BANDS; ++b) {
      mbar_init(&bfull[b], PR_NPW);
      mbar_init(&bempty[b], 1);
      if constexpr (PAIR) mbar_init(&pbfull[b], 1);
    }
    if (bias_on) mbar_init(bbias, 1);
    if (ALIGN && g.raw)
      for (int r = 0; r < PR_RAW_SLOTS; ++r) {
        mbar_init(&rfull[r], 1);
        mbar_init(&rempty[r], PR_NPW);
      }
    for (int a = 0; a < PR_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 2 * PR_NEPI : PR_NEPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&bmap) : "memory");
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {  // unit block scales
    uint32_t ones[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) ones[i] = 0x7F7F7F7Fu;
    tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + SF_COL, ones);
    if constexpr (BIAS) {  // every lane quarter holds the B scales of all N rows (n % 32, column n / 32)
#pragma unroll
      for (int i = 0; i < 16; ++i) ones[i] = PR_BIAS_SF;
      tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + SF_BIAS, ones);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync_all();  // both CTAs' barriers and scale factors exist before any remote access
  else
    __syncthreads();
  tc_fence_after();
  pdl_entry();

  if (warp == 0) {
    // ------------------------------------------------ weights, once (PAIR: this CTA's half of the filters)
    const int nkb_ld = g.nkb_ld ? g.nkb_ld : g.nkb;
    if (lane == 0 && !TW) {
      mbar_expect_tx(bres, (uint32_t)nkb_ld * BNH * 128);
      for (int a = 0; a < nkb_ld; ++a) tma_load_2d(sb + a * BNH * 128, &bmap, bres, a * 128, (int)rank * BNH);
    }
    if (bias_on) {
      // each filter's threshold block at K = kk .. kk + 63 of its weight row
      // (128-byte swizzled atoms: 16-byte chunk c of row n at c ^ (n & 7))
      mbar_wait(bres, 0);
      const int a = g.kk >> 8, ch = ((g.kk & 255) >> 1) >> 4;
      const int64_t kmax = g.kk + 1;
      for (int n = lane; n < BN; n += 32) {
        const int64_t b = filter_bias(g.thresh, g.ge, n, g.F, kmax - 1);
        uint4 b0, b1;
        pr_bias_bytes(b, b0, b1);
        uint8_t* row = sb + a * BNH * 128 + (n >> 3) * 1024 + (n & 7) * 128;
        *reinterpret_cast<uint4*>(row + ((ch ^ (n & 7)) << 4)) = b0;
        *reinterpret_cast<uint4*>(row + (((ch + 1) ^ (n & 7)) << 4)) = b1;
      }
      for (int i = lane; i < 4096 / 16; i += 32)  // the threshold block's +1 operand
        reinterpret_cast<uint4*>(sones)[i] = make_uint4(0x22222222u, 0x22222222u, 0x22222222u, 0x22222222u);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bbias);
    }
  } else if (ALIGN && warp == 3 && g.raw) {
    // ------------------------------------------------ input loader (ALIGN)
    // The tile's input pixels (rows y0 - pad .. y0 + 128/W - 1 + pad of one
    // image, clamped to the image: one contiguous range) arrive by 1-D bulk
    // copy into a ring of PR_RAW_SLOTS staging slots that the producer warps
    // release one by one (a per-tile named barrier among the producers, with
    // one of them issuing the copies, held every producer to the slowest:
    // ncu put the producers' top stall on that barrier).  Staging row b holds
    // band pixel b.
    if (lane == 0) {
      const uint32_t raw_bytes = (uint32_t)g.Rb * (uint32_t)g.sstride * 4u;
      int rs = 0;
      uint32_t rph = 0;
      for (int64_t t = t_first; t < tiles; t += t_step) {
        mbar_wait_sleep(&rempty[rs], rph ^ 1, B2_PR_SLEEP_NS);  // (polling cost ~180 issue slots per tile)
        const int64_t p0 = t * BM, n = p0 / g.HW;
        const int64_t lo = p0 - n * g.HW - (int64_t)g.pad * g.W, hi = lo + g.Rb;
        const int64_t l0 = lo < 0 ? 0 : lo, h0 = hi > g.HW ? g.HW : hi;
        const uint32_t bytes = (uint32_t)((h0 - l0) * g.sstride * 4);
        mbar_expect_tx(&rfull[rs], bytes);
        bulk_g2s_pr(sraw + (size_t)rs * raw_bytes + (size_t)(l0 - lo) * g.sstride * 4, g.x + (n * g.HW + l0) * g.sstride,
                    bytes, &rfull[rs]);
        if (++rs == PR_RAW_SLOTS) rs = 0, rph ^= 1;
      }
    }
  } else if (warp == 1 && PAIR && rank == 1) {
    // ------------------------------------------------ relay (PAIR, CTA 1): my band is full
    if (lane == 0) {
      const uint32_t peer = cluster_map(smem_u32(pbfull), 0);
      int slot = 0;
      uint32_t bph = 0;
      for (int64_t t = t_first; t - rank < tiles; t += t_step) {
        mbar_wait(&bfull[slot], bph);
        mbar_arrive_remote(peer + 8u * (uint32_t)slot);
        if (++slot == PR_BANDS) slot = 0, bph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (PAIR: CTA 0 issues for both)
    // B2_PR_WARP_ISSUE: the whole warp runs the issue loop (descriptors are
    // warp-uniform, so they stay in uniform registers) and one elected lane
    // issues; a lone lane-0 thread re-broadcast every descriptor (R2UR) per
    // MMA, and under epilogue load that chain outlasted the 64-cycle MMA
    // (row-aligned kernels; the virtual-grid 256-column conv3 measured slower
    // with it: 1.83 vs 1.69 ms)
    constexpr bool WI = (ALIGN || B2_PR_WI_ALL) && B2_PR_WARP_ISSUE;
    if (WI || lane == 0) {
      // descriptor offsets of every MMA of a tile, once: (window cell, K chunk)
      // -> band plane + row shift for A, weight atom + 32-byte step for B
      int nmma = 0;
      for (int cy = 0; cy < g.kh; ++cy)
        for (int cx = 0; cx < g.kw; ++cx) {
          // band row of tile row 0 (ALIGN: copy cx, cy rows of W down)
          const int off = ALIGN ? (cy << g.wshift) : g.band0 + (cy - g.pad) * g.Wp + (cx - g.pad);
          const int plane0 = ALIGN ? cx * g.P : 0;
          const int cell = cy * g.kw + cx;
          for (int kc = 0; kc < g.kmmas; ++kc, ++nmma) {
            const int k = cell * g.P * 32 + kc * 64;  // K element
            if (lane == 0) soff[nmma] = make_uint2(((uint32_t)(plane0 + 2 * kc) * plane_bytes + (uint32_t)off * 16u) >> 4,
                                    TW ? (uint32_t)(k >> 3)
                                       : (uint32_t)((k >> 8) * BNH * 128 + ((k & 255) >> 6) * 32) >> 4);
          }
        }
      if constexpr (WI) __syncwarp();
      mbar_wait(bres, 0);
      if (bias_on) mbar_wait(bbias, 0);
      const uint64_t ones_desc = noswz_desc(smem_u32(sones), 2048);
      const uint32_t bias_bo = BIAS ? (uint32_t)((g.kk >> 8) * BNH * 128 + ((g.kk & 255) >> 6) * 32) >> 4 : 0u;
      int slot = 0, acc = 0;
      uint32_t bph = 0, aph = 0;
      const uint64_t bdesc0 = sw128_desc(smem_u32(sb));
      const uint32_t b_lo = (uint32_t)bdesc0, b_hi = (uint32_t)(bdesc0 >> 32);
      const uint32_t tm = WI ? __shfl_sync(0xffffffffu, tmem, 0) : tmem;  // warp-uniform TMEM base
#ifdef B2_PR_TIMING
      long long c_band = 0, c_acc = 0, c_issue = 0, c_t0 = clock64();
#endif
      for (int64_t t = t_first; t - rank < tiles; t += t_step) {
#ifdef B2_PR_TIMING
        long long c0 = clock64();
#endif
        mbar_wait(&bfull[slot], bph);
        if constexpr (PAIR) mbar_wait(&pbfull[slot], bph);
#ifdef B2_PR_TIMING
        long long c1 = clock64();
#endif
        mbar_wait(&tempty[acc], aph ^ 1);
#ifdef B2_PR_TIMING
        long long c2 = clock64();
        c_band += c1 - c0, c_acc += c2 - c1;
#endif
        tc_fence_after();
        // descriptors as (lo + offset, hi): the offsets only touch the 14-bit
        // start-address field; with tm broadcast from lane 0 every operand is
        // warp-uniform and the issue sequence stays in uniform registers
        const uint32_t d = tm + acc * ACC_COLS;
        const uint64_t adesc0 = noswz_desc(smem_u32(sband + slot * g.band_bytes), plane_bytes);
        const uint32_t a_lo = (uint32_t)adesc0, a_hi = (uint32_t)(adesc0 >> 32);
        auto dsc = [](uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; };
        const bool leader = pr_elect<WI>();
        if (leader) {
        if constexpr (KH > 0) {
          constexpr int PAD = KH / 2;
#pragma unroll
          for (int cy = 0; cy < KH; ++cy)
#pragma unroll
            for (int cx = 0; cx < KH; ++cx)
#pragma unroll
              for (int kc = 0; kc < KMMAS; ++kc) {
                const int cell = cy * KH + cx;
                const int k = (cell * KMMAS + kc) * 64;  // K element (c = 32 * 2 * KMMAS)
                const uint32_t off = ALIGN ? (uint32_t)(cy << g.wshift) : (uint32_t)(g.band0 + (cy - PAD) * g.Wp + (cx - PAD));
                const uint32_t plane = ALIGN ? (uint32_t)(cx * 2 * KMMAS + 2 * kc) : (uint32_t)(2 * kc);
                const uint32_t ao = (plane * plane_bytes + off * 16u) >> 4;
                const uint32_t bo = (uint32_t)((k >> 8) * BNH * 128 + ((k & 255) >> 6) * 32) >> 4;
                if constexpr (TW)
                  tc_mma_f4_ts(d, tm + PR_TW_COL + (uint32_t)(k >> 3), dsc(a_lo + ao, a_hi), IDESC, tm + SF_COL,
                               tm + SF_COL + 4, (cell | kc) ? 1u : 0u);
                else if constexpr (PAIR)
                  tc_mma_f4_pair(d, dsc(a_lo + ao, a_hi), dsc(b_lo + bo, b_hi), IDESC, tm + SF_COL, tm + SF_COL + 4,
                                 (cell | kc) ? 1u : 0u);
                else
                  tc_mma_f4(d, dsc(a_lo + ao, a_hi), dsc(b_lo + bo, b_hi), IDESC, tm + SF_COL, tm + SF_COL + 4,
                            (cell | kc) ? 1u : 0u);
              }
        } else {
          for (int i = 0; i < nmma; ++i) {
            const uint2 o = soff[i];
            if constexpr (TW)
              tc_mma_f4_ts(d, tm + PR_TW_COL + o.y, dsc(a_lo + o.x, a_hi), IDESC, tm + SF_COL, tm + SF_COL + 4,
                           i ? 1u : 0u);
            else if constexpr (PAIR)
              tc_mma_f4_pair(d, dsc(a_lo + o.x, a_hi), dsc(b_lo + o.y, b_hi), IDESC, tm + SF_COL, tm + SF_COL + 4,
                             i ? 1u : 0u);
            else
              tc_mma_f4(d, dsc(a_lo + o.x, a_hi), dsc(b_lo + o.y, b_hi), IDESC, tm + SF_COL, tm + SF_COL + 4,
                        i ? 1u : 0u);
          }
        }
        if (bias_on)
          tc_mma_f4(d, ones_desc, dsc(b_lo + bias_bo, b_hi), IDESC, tm + SF_COL, tm + SF_BIAS, 1u);
        }
#ifdef B2_PR_TIMING
        c_issue += clock64() - c2;
#endif
        if (!leader) {
        } else if constexpr (PAIR) {
          tc_commit_pair(&bempty[slot]);
          tc_commit_pair(&tfull[acc]);
        } else {
          tc_commit(&bempty[slot]);
          tc_commit(&tfull[acc]);
        }
        if (++slot == PR_BANDS) slot = 0, bph ^= 1;
        if (++acc == PR_ACC) acc = 0, aph ^= 1;
      }
#ifdef B2_PR_TIMING
      if (blockIdx.x < 3 && lane == 0)
        printf("cta %d: total %lld  wait band %lld  wait acc %lld  issue %lld  tiles %lld\n", blockIdx.x,
               clock64() - c_t0, c_band, c_acc, c_issue, (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
#endif
    }
  } else if (warp >= 4 && warp < EPI0) {
    // ------------------------------------------------ band producers
    if constexpr (BYTEIN) {
      // byte-BN first layer: one band row per thread per tile; plane 0 =
      // the pixel's thresholded channel bits (<= 8) as e2m1, plane 1 = 0
      const int pt = (warp - 4) * 32 + lane;  // 0 .. 255
      int32_t tin[8];
      bool gin[8];
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        tin[ch] = ch < g.cin ? __ldg(g.th_in + ch) : 0;
        gin[ch] = ch < g.cin ? __ldg(g.ge_in + ch) != 0 : true;
      }
      const uint32_t cmask = (1u << g.cin) - 1u;
      for (int sl = 0; sl < PR_BANDS; ++sl)  // the zero planes, once
        for (int b = pt; b < g.R8; b += 32 * PR_NPW)
          *reinterpret_cast<uint4*>(sband + sl * g.band_bytes + plane_bytes + (size_t)b * 16) = make_uint4(0, 0, 0, 0);
      int slot = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t v0 = t * BM - g.band0;
        uint32_t bits[2] = {0, 0};
        bool ok[2] = {false, false};
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int b = pt + i * 32 * PR_NPW;
          const int64_t v = v0 + b;
          if (b < g.R8 && v >= 0 && v < g.Vtotal) {
            int64_t n;
            int y, x;
            vsplit(g, v, n, y, x);
            if (y < g.H && x < g.W) {
              ok[i] = true;
              const uint8_t* px = g.xb + ((n * g.H + y) * g.W + x) * g.cin;
#pragma unroll
              for (int ch = 0; ch < 8; ++ch)
                if (ch < g.cin) bits[i] |= (thr_bit((int32_t)__ldg(px + ch), tin[ch], gin[ch]) ? 1u : 0u) << ch;
            }
          }
        }
        mbar_wait_suspend(&bempty[slot], ph ^ 1);
        uint8_t* band = sband + slot * g.band_bytes;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int b = pt + i * 32 * PR_NPW;
          if (b < g.R8) {
            uint32_t o[4];
            widen_f4m(bits[i], ok[i] ? cmask : 0u, o);
            *reinterpret_cast<uint4*>(band + (size_t)b * 16) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bfull[slot]);
        if (++slot == PR_BANDS) slot = 0, ph ^= 1;
      }
    } else if constexpr (ALIGN) {
      // row-aligned tiles: unit = (band row b, 4-word group); the input pixel
      // of band row b (input row y0 - pad + b / W, column b % W) is expanded
      // once and stored into each copy dx at row b - dx + pad (the copy's
      // column x' = x - dx + pad must lie in the row).  Copy rows that no
      // pixel maps to (x' + dx - pad outside the row) stay zero from the
      // one-time clear below; rows above / below the image are stored as
      // zeros.  The next tile's loads are issued before this tile's band is
      // written (register double buffer), so their latency overlaps.
      constexpr int UMAX = 2;
      const int pt = (warp - 4) * 32 + lane;  // 0 .. 255
      const int groups = KH > 0 ? KMMAS / 2 : g.P / 4;  // compile-time for the 3x3 kernels (no division below)
      const int units = g.Rb * groups;
      const int kwc = KH > 0 ? KH : g.kw;
      const int wmask = (1 << g.wshift) - 1;
      for (int i = pt; i < PR_BANDS * g.band_bytes / 16; i += 32 * PR_NPW)
        reinterpret_cast<uint4*>(sband)[i] = make_uint4(0, 0, 0, 0);
      asm volatile("bar.sync 2, %0;" ::"n"(32 * PR_NPW) : "memory");  // the clear lands before any copy row is stored
      if (!g.raw) {
      // no room for the staging ring (256 filters: 160 KB of weights): each
      // producer loads the next tile's pixels into registers before storing
      // the current band (register double buffer)
      auto load_tile = [&](int64_t t, uint4 (&w)[UMAX], bool (&ok)[UMAX]) {
        const int64_t n = t / (g.HW / BM);
        const int y0 = (int)(((t - n * (g.HW / BM)) * BM) >> g.wshift);
        const uint32_t* img = g.x + n * g.HW * g.sstride;
#pragma unroll
        for (int i = 0; i < UMAX; ++i) {
          const int u = pt + i * 32 * PR_NPW;
          ok[i] = false;
          w[i] = make_uint4(0, 0, 0, 0);
          if (t < tiles && u < units) {
            const int b = u / groups, grp = u - b * groups;
            const int y = y0 - g.pad + (b >> g.wshift);
            if ((unsigned)y < (unsigned)g.H) {
              ok[i] = true;
              w[i] = __ldg(reinterpret_cast<const uint4*>(img + ((int64_t)(y << g.wshift) + (b & wmask)) * g.sstride +
                                                          4 * grp));
            }
          }
        }
      };
      int slot = 0;
      uint32_t ph = 0;
      uint4 wa[UMAX], wb[UMAX];
      bool oka[UMAX], okb[UMAX];
      load_tile(t_first, wa, oka);
      auto tile = [&](int64_t t, uint4 (&wc)[UMAX], bool (&okc)[UMAX], uint4 (&wn)[UMAX], bool (&okn)[UMAX]) {
        load_tile(t + t_step, wn, okn);
        B2_PR_PROD_WAIT(&bempty[slot], ph ^ 1);
        uint8_t* band = sband + slot * g.band_bytes;
#pragma unroll
        for (int i = 0; i < UMAX; ++i) {
          const int u = pt + i * 32 * PR_NPW;
          if (u < units) {
            const int b = u / groups, grp = u - b * groups;
            const int x = b & wmask;
            uint32_t o[16];
            widen_f4(wc[i].x, okc[i], o);
            widen_f4(wc[i].y, okc[i], o + 4);
            widen_f4(wc[i].z, okc[i], o + 8);
            widen_f4(wc[i].w, okc[i], o + 12);
#pragma unroll 3
            for (int dx = 0; dx < kwc; ++dx) {
              const int xp = x - dx + g.pad;
              if ((unsigned)xp < (unsigned)(wmask + 1)) {
                uint8_t* row = band + (size_t)(dx * g.P + 4 * grp) * plane_bytes + (size_t)(b - dx + g.pad) * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  *reinterpret_cast<uint4*>(row + (size_t)j * plane_bytes) =
                      make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
              }
            }
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bfull[slot]);
        if (++slot == PR_BANDS) slot = 0, ph ^= 1;
      };
      for (int64_t t = t_first; t - rank < tiles; t += 2 * t_step) {
        tile(t, wa, oka, wb, okb);
        if (t + t_step - rank < tiles) tile(t + t_step, wb, okb, wa, oka);
      }
      } else {
      // input pixels from the loader warp's staging ring
      const uint32_t raw_bytes = (uint32_t)g.Rb * (uint32_t)g.sstride * 4u;
      int slot = 0, rslot = 0;
      uint32_t ph = 0, rph = 0;
#ifdef B2_PR_TIMING
      long long p_wait = 0, p_work = 0, p_sync = 0, p_raw = 0, p_t0 = clock64();
#endif
      // tile t = image t / tpi, first row (t % tpi) * BM / W: stepped
      // incrementally (a 64-bit division per tile was ~25 instructions)
      const int tpi = (int)(g.HW / BM), trows = BM >> g.wshift;
      const int step_r = (int)(t_step % tpi);
      int tr = (int)(t_first % tpi);
      for (int64_t t = t_first; t - rank < tiles; t += t_step) {
        const int y0 = tr * trows;
        if ((tr += step_r) >= tpi) tr -= tpi;
        const bool tvalid = t < tiles;
#ifdef B2_PR_TIMING
        long long r0 = clock64();
#endif
        if (tvalid) mbar_wait(&rfull[rslot], rph);
#ifdef B2_PR_TIMING
        p_raw += clock64() - r0;
#endif
        const uint8_t* raw = sraw + (size_t)rslot * raw_bytes;
        uint4 wc[UMAX];
        bool okc[UMAX];
#pragma unroll
        for (int i = 0; i < UMAX; ++i) {
          const int u = pt + i * 32 * PR_NPW;
          okc[i] = false;
          wc[i] = make_uint4(0, 0, 0, 0);
          if (tvalid && u < units) {
            const int b = u / groups, grp = u - b * groups;
            const int y = y0 - g.pad + (b >> g.wshift);
            if ((unsigned)y < (unsigned)g.H) {
              okc[i] = true;
              wc[i] = *reinterpret_cast<const uint4*>(raw + (size_t)b * g.sstride * 4 + 16 * grp);
            }
          }
        }
        __syncwarp();
        if (tvalid && lane == 0) mbar_arrive(&rempty[rslot]);  // the staging slot may be refilled
#ifdef B2_PR_TIMING
        long long q0 = clock64();
#endif
        B2_PR_PROD_WAIT(&bempty[slot], ph ^ 1);
#ifdef B2_PR_TIMING
        p_wait += clock64() - q0;
#endif
        uint8_t* band = sband + slot * g.band_bytes;
#pragma unroll
        for (int i = 0; i < UMAX; ++i) {
          const int u = pt + i * 32 * PR_NPW;
#ifdef B2_X_NOSTORE  // experiment: producers skip the band stores
          if (u < units && wc[i].x == 0x12345678u) {
#else
          if (u < units) {
#endif
            const int b = u / groups, grp = u - b * groups;
            const int x = b & wmask;
            uint32_t o[16];
            widen_f4(wc[i].x, okc[i], o);
            widen_f4(wc[i].y, okc[i], o + 4);
            widen_f4(wc[i].z, okc[i], o + 8);
            widen_f4(wc[i].w, okc[i], o + 12);
#pragma unroll 3
            for (int dx = 0; dx < kwc; ++dx) {
              const int xp = x - dx + g.pad;
              if ((unsigned)xp < (unsigned)(wmask + 1)) {
                uint8_t* row = band + (size_t)(dx * g.P + 4 * grp) * plane_bytes + (size_t)(b - dx + g.pad) * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  *reinterpret_cast<uint4*>(row + (size_t)j * plane_bytes) =
                      make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
              }
            }
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bfull[slot]);
        if (++slot == PR_BANDS) slot = 0, ph ^= 1;
        if (++rslot == PR_RAW_SLOTS) rslot = 0, rph ^= 1;
      }
#ifdef B2_PR_TIMING
      p_work = clock64() - p_t0 - p_wait;
      if (blockIdx.x < 2 && (pt == 0 || pt == 255))
        printf("producer cta %d t%d: total %lld  wait slot %lld  sync %lld  raw %lld  other %lld\n", blockIdx.x, pt,
               clock64() - p_t0, p_wait, p_sync, p_raw, p_work - p_sync - p_raw);
#endif
      }  // g.raw
    } else {
    // each thread owns up to UMAX (band row, 4-word group) units per tile;
    // a tile's loads are issued before waiting for its band slot
    constexpr int UMAX = 2;
    const int pt = (warp - 4) * 32 + lane;  // 0 .. 255
    const int groups = KH > 0 ? KMMAS / 2 : g.P / 4;  // 4-word groups per pixel
    const int units = g.R8 * groups;
    int slot = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int64_t v0 = t * BM - g.band0;
      uint4 w[UMAX];
      bool ok[UMAX];
#pragma unroll
      for (int i = 0; i < UMAX; ++i) {
        const int u = pt + i * 32 * PR_NPW;
        ok[i] = false;
        w[i] = make_uint4(0, 0, 0, 0);
        if (u < units) {
          const int b = u / groups, grp = u - b * groups;
          const int64_t v = v0 + b;
          if (v >= 0 && v < g.Vtotal) {
            int64_t n;
            int y, x;
            vsplit(g, v, n, y, x);
            if (y < g.H && x < g.W) {
              ok[i] = true;
              w[i] = __ldg(reinterpret_cast<const uint4*>(g.x + ((n * g.H + y) * g.W + x) * g.sstride + 4 * grp));
            }
          }
        }
      }
      mbar_wait_suspend(&bempty[slot], ph ^ 1);
      uint8_t* band = sband + slot * g.band_bytes;
#pragma unroll
      for (int i = 0; i < UMAX; ++i) {
        const int u = pt + i * 32 * PR_NPW;
        if (u < units) {
          const int b = u / groups, grp = u - b * groups;
          uint32_t o[16];
          widen_f4(w[i].x, ok[i], o);
          widen_f4(w[i].y, ok[i], o + 4);
          widen_f4(w[i].z, ok[i], o + 8);
          widen_f4(w[i].w, ok[i], o + 12);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(band + (size_t)(4 * grp + j) * plane_bytes + (size_t)b * 16) =
                make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bfull[slot]);
      if (++slot == PR_BANDS) slot = 0, ph ^= 1;
    }
    }
  } else if (TW && warp >= EPI0) {
    // ------------------------------------------------ epilogue, filters on TMEM lanes (TW)
    static_assert(!TW || SF_COL + 16 <= PR_TW_COL, "TMEM: accumulators, scales, weights");
    const int q = warp & 3;                 // lane quarter: filters 32 q .. 32 q + 31
    const int hh = (warp - EPI0) >> 2;      // pixels 64 hh .. 64 hh + 63 of the tile
    const int f = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    {
      // this warp's half of its 32 filter rows' weights -> TMEM (A operand)
      const int half = (g.wt_words + 31) / 32 * 16, j0 = hh * half, j1 = min(g.wt_words, j0 + half);
      const uint32_t* wrow = g.wt + (size_t)f * g.wt_stride;
      for (int j = j0; j < j1; j += 16) {
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = (f < g.F && j + i < j1) ? __ldg(wrow + j + i) : 0u;
        tmem_st16(lane_base + PR_TW_COL + j, v);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bres);
    }
    float mul = 0.f, add = -1.f;  // filters past F: bit 0 (the (mul, add) of stage_thresholds)
    bool ge = true;
    if (f < g.F) {
      const int32_t th = __ldg(g.thresh + f);
      ge = __ldg(g.ge + f) != 0;
      mul = ge ? 1.f : -1.f;
      add = (float)(ge ? -th : th);
    }
    const uint32_t gm = __ballot_sync(0xffffffffu, ge);  // OR-pool (ge) / AND-pool (le) filters
    const bool store_q = q < (g.wlim ? g.wlim : g.ldo32);
    const int wmask = (1 << g.wshift) - 1;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = t_first; t < tiles; t += t_step) {
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      uint32_t va[32], vb[32];
      const uint32_t ta = lane_base + acc * ACC_COLS + hh * 64;
      tmem_ld32(ta, va);
      tmem_ld32(ta + 32, vb);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
#ifdef B2_X_NOEPI  // experiment: the epilogue only drains
      if (va[0] != 0x12345678u) { if (++acc == PR_ACC) acc = 0, aph ^= 1; continue; }
#endif
      // sign words: lane j ends with the 32-filter word of pixel j (wa) and
      // pixel 32 + j (wb) of this warp's 64
      uint32_t wa = 0, wb = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        // bit = sign bit clear, as thr_word (-0 counts as negative)
        const uint32_t ba = __ballot_sync(0xffffffffu, (int)__float_as_uint(__fmaf_rn(__uint_as_float(va[j]), mul, add)) >= 0);
        const uint32_t bb = __ballot_sync(0xffffffffu, (int)__float_as_uint(__fmaf_rn(__uint_as_float(vb[j]), mul, add)) >= 0);
        wa = lane == j ? ba : wa;
        wb = lane == j ? bb : wb;
      }
      const int64_t pix = t * BM + hh * 64 + lane;  // pixel of wa (wb: + 32)
      if (!g.pool) {
        if (store_q) {
          g.out_bits[pix * g.ldo32 + q] = wa;
          g.out_bits[(pix + 32) * g.ldo32 + q] = wb;
        }
      } else {
        // 2x2/2 pool: vertical partner in wb (W = 32) or lane ^ W (W <= 16),
        // horizontal partner lane ^ 1; the top-left lane of each window stores
        const int x = lane & wmask;
        const int wp = (1 << g.wshift) >> 1;
        auto store_pooled = [&](uint32_t o, uint32_t an, int64_t px, bool top) {
          o |= __shfl_xor_sync(0xffffffffu, o, 1);
          an &= __shfl_xor_sync(0xffffffffu, an, 1);
          if (store_q && top && !(x & 1)) {
            const int ty = (int)(px - t * BM) >> g.wshift;  // row within the tile (tiles are whole row pairs)
            g.out_bits[(t * (BM / 4) + (ty >> 1) * wp + (x >> 1)) * g.ldo32 + q] = (o & gm) | (an & ~gm);
          }
        };
        if (g.wshift == 5) {
          store_pooled(wa | wb, wa & wb, pix, true);
        } else {
          const int vs = 1 << g.wshift;
          const bool top = !(lane & vs);
          const uint32_t wa2 = __shfl_xor_sync(0xffffffffu, wa, vs), wb2 = __shfl_xor_sync(0xffffffffu, wb, vs);
          store_pooled(wa | wa2, wa & wa2, pix, top);
          store_pooled(wb | wb2, wb & wb2, pix + 32, top);
        }
      }
      if (++acc == PR_ACC) acc = 0, aph ^= 1;
    }
  } else if (warp >= EPI0) {
    // ------------------------------------------------ epilogue
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int et = (warp - EPI0) * 32 + lane;
    constexpr int ECH = (BN / 32) / (PR_NEPI / 4);  // 32-column chunks per epilogue warp
    const int c0 = ((warp - EPI0) >> 2) * ECH;    // first chunk of this warp
    {
      Args ga{};
      ga.N = g.F;
      ga.thresh = g.thresh;
      ga.ge = g.ge;
      stage_thresholds<true>(ga, 0, BN, et, 32 * PR_NEPI, lane, sthr, sgm);
    }
    epi_bar<PR_NEPI>();
    const int64_t wlim = g.wlim ? g.wlim : g.ldo32;
    // sign word of accumulator chunk ch: BIAS folded the threshold into the
    // accumulator (bit = sign ^ le), otherwise the (mul, add) table
    auto epi_word = [&](const uint32_t (&v)[32], int ch) -> uint32_t {
      if (bias_on)
        return sign_word(v) ^ sgm[ch];
      else
        return thr_word<true>(v, sthr + ch * 16);
    };
    int acc = 0;
    uint32_t aph = 0;
    uint32_t it = 0;  // tiles done by this CTA (ALIGN pool buffer parity)
    (void)it;
    // release accumulator `a`: CTA 0's barrier (PAIR: both CTAs' epilogues count)
    const uint32_t peer_tempty = PAIR && rank ? cluster_map(smem_u32(tempty), 0) : 0u;
    auto release_acc = [&](int a) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && rank)
          mbar_arrive_remote(peer_tempty + 8u * (uint32_t)a);
        else
          mbar_arrive(&tempty[a]);
      }
    };
    for (int64_t t = t_first; t - rank < tiles; t += t_step) {
      const bool tv = t < tiles;  // PAIR: the last pair's second half may lie past the end
#if B2_PR_EPI_SUSPEND
      mbar_wait_suspend(&tfull[acc], aph);
#else
      mbar_wait(&tfull[acc], aph);
#endif
      tc_fence_after();
      uint32_t words[ECH];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * ACC_COLS + c0 * 32;
      if constexpr (ECH <= 2) {
        // every chunk's load in flight at once, one wait: the accumulator goes
        // back to the MMA after a single TMEM round trip
        uint32_t v[ECH][32];
#pragma unroll
        for (int c = 0; c < ECH; ++c) tmem_ld32(ta + c * 32, v[c]);
        tmem_wait_ld();
        release_acc(acc);
#pragma unroll
        for (int c = 0; c < ECH; ++c) words[c] = epi_word(v[c], (c0 + c));
      } else if (ECH == 4 && PR_ACC == 1 && bias_on && B2_PR_DRAIN2) {
        // bias fold: a chunk is its sign word at once, so two TMEM round
        // trips with the first pair's words in between release the single
        // 256-column accumulator (conv3's MMA thread waited 29 % for it)
        uint32_t va[32], vb[32];
        tmem_ld32(ta, va);
        tmem_ld32(ta + 32, vb);
        tmem_wait_ld();
        words[0] = epi_word(va, c0);
        words[1] = epi_word(vb, (c0 + 1));
        tmem_ld32(ta + 64, va);
        tmem_ld32(ta + 96, vb);
        tmem_wait_ld();
        release_acc(acc);
        words[2] = epi_word(va, (c0 + 2));
        words[3] = epi_word(vb, (c0 + 3));
      } else if constexpr (ECH == 4 && PR_ACC == 1 && B2_TMEM_STAGE) {
        // the single 256-column accumulator (BNT = 256): stage the first two
        // chunks in spare TMEM columns (past the accumulator and the scale
        // factors), load the last two, release — three TMEM round trips —
        // then threshold from registers / spare (MMA-thread timing: conv3
        // waited 42 % of its time for the accumulator)
        const uint32_t spare = tmem + ((uint32_t)(q * 32) << 16) + 288 + ((warp - EPI0) >> 2) * 64;
        static_assert(SF_COL + 16 <= 288 && 288 + 2 * 64 <= 512, "spare TMEM columns");
        uint32_t va[32], vb[32];
        tmem_ld32(ta, va);
        tmem_ld32(ta + 32, vb);
        tmem_wait_ld();
        tmem_st32(spare, va);
        tmem_st32(spare + 32, vb);
        tmem_wait_st();
        tmem_ld32(ta + 64, va);
        tmem_ld32(ta + 96, vb);
        tmem_wait_ld();
        release_acc(acc);
        words[2] = epi_word(va, (c0 + 2));
        words[3] = epi_word(vb, (c0 + 3));
        tmem_ld32(spare, va);
        tmem_ld32(spare + 32, vb);
        tmem_wait_ld();
        words[0] = epi_word(va, c0);
        words[1] = epi_word(vb, (c0 + 1));
      } else {
      // software-pipelined: chunk c + 1 is in flight while chunk c is thresholded
      uint32_t va[32], vb[32];
      tmem_ld32(ta, va);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < ECH; ++c) {
        uint32_t(&v)[32] = (c & 1) ? vb : va;
        uint32_t(&vn)[32] = (c & 1) ? va : vb;
        if (c + 1 < ECH) tmem_ld32(ta + (c + 1) * 32, vn);
        words[c] = epi_word(v, (c0 + c));
        if (c + 1 < ECH) tmem_wait_ld();
        if (c + 2 == ECH) {  // every chunk is in registers: return the accumulator before the last one's math
          release_acc(acc);
        }
      }
      }
      if constexpr (ALIGN) {
        const int64_t pix = t * BM + r;  // tiles cover whole images: every row is a pixel
        if (!g.pool) {
          uint32_t* o = g.out_bits + pix * g.ldo32;
          if (tv)
#pragma unroll
          for (int c = 0; c < ECH; ++c)
            if (c0 + c < wlim) o[c0 + c] = words[c];
        } else {
          // 2x2/2 pool inside the tile: OR / AND of the horizontal pair by
          // shuffle, then of the vertical pair (row r + W) through shared
          // memory (double-buffered by tile parity: one barrier per tile)
          uint2* sp = spool + (size_t)(it & 1) * BM * (BN / 32);
#pragma unroll
          for (int c = 0; c < ECH; ++c) {
            const uint32_t w1 = __shfl_xor_sync(0xffffffffu, words[c], 1);
            sp[(c0 + c) * BM + r] = make_uint2(words[c] | w1, words[c] & w1);  // [column word][row]: no bank conflicts
          }
          epi_bar<PR_NEPI>();
          const int ty = r >> g.wshift, x = r & ((1 << g.wshift) - 1);
          if (tv && !(ty & 1) && !(x & 1)) {
            // a tile is whole row pairs of one image: its pooled sites are
            // the BM / 4 consecutive sites from t BM / 4
            const int wp = (1 << g.wshift) >> 1;
            uint32_t* o = g.out_bits + (t * (BM / 4) + (ty >> 1) * wp + (x >> 1)) * g.ldo32;
#pragma unroll
            for (int c = 0; c < ECH; ++c) {
              const uint2 a = sp[(c0 + c) * BM + r], b = sp[(c0 + c) * BM + r + (1 << g.wshift)];
              const uint32_t gm = sgm[c0 + c];
              if (c0 + c < wlim) o[c0 + c] = ((a.x | b.x) & gm) | ((a.y & b.y) & ~gm);
            }
          }
        }
        ++it;
      } else {
      const int64_t v = t * BM + r;
      if (v < g.Vtotal) {
        int64_t n;
        int y, x;
        vsplit(g, v, n, y, x);
        if (y < g.H && x < g.W) {
          uint32_t* o = g.out_bits + ((n * g.H + y) * g.W + x) * g.ldo32;
#pragma unroll
          for (int c = 0; c < ECH; ++c)
            if (c0 + c < wlim) o[c0 + c] = words[c];
        }
      }
      }
      if (++acc == PR_ACC) acc = 0, aph ^= 1;
    }
  }
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync_all();  // no CTA leaves while its peer can still touch its shared or tensor memory
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Byte-input first-layer weights for the padded-row kernel: per window cell
// 64 K elements — the cell's c (<= 8) channel bits as e2m1 in the first 32
// (widen_f4 order), then 32 zeros — so each cell is one K=64 MMA reading
// the band's data plane and zero plane.  Packed rows hold K = cells * c
// bits in (dy, dx, c) order (the reference's layout).
__global__ void k_expand_f4_cells(const uint64_t* __restrict__ w, int64_t rows, int64_t wpl, int cells, int c,
                                  int64_t row_words, uint32_t* __restrict__ out) {
  pdl_entry();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * row_words) return;
  const int64_t r = t / row_words;
  const int o = (int)(t - r * row_words);
  const int cell = o >> 3, q = o & 7;
  uint32_t word = 0;
  if (cell < cells && q < 4) {
    const int64_t k0 = (int64_t)cell * c;  // first bit of the cell
    const uint64_t* line = w + r * wpl;
    uint32_t bits = (uint32_t)(line[k0 >> 6] >> (k0 & 63));
    if ((k0 & 63) + c > 64) bits |= (uint32_t)(line[(k0 >> 6) + 1] << (64 - (k0 & 63)));
    const uint32_t valid = (1u << c) - 1u;
    word = (0xAAAAAAAAu ^ ((bits << (3 - q)) & 0x88888888u)) & (((valid >> q) & 0x11111111u) * 0xFu);
  }
  out[t] = word;
}

// raw_bytes > 0 (ALIGN): the staging ring and its barriers (after the pool
// exchange, which only pooled / pair launches lay out); bias: the threshold
// block's barrier and +1 operand (after the MMA offset table)
template <int BNT>
inline int padrow_smem_bytes(int nkb, int band_bytes, int nbands = pr_bands<BNT>(), bool pool_buf = false,
                             bool pair = false, int raw_bytes = 0, bool bias = false) {
  return nkb * (pair ? BNT / 2 : BNT) * 128 + nbands * band_bytes + BNT / 2 * 16 + BNT / 8 +
         8 * (1 + 2 * PR_BANDS_MAX + 2 * pr_acc<BNT>()) + 16 + 8 * 128 +  // MMA offset table (<= 128)
         (bias ? 16 + 128 + 4096 : 0) +
         (pool_buf || pair ? 2 * BM * (BNT / 32) * 8 : 0) + (pair || raw_bytes ? 8 * PR_BANDS_MAX : 0) +
         (raw_bytes ? 16 * PR_RAW_SLOTS + 16 + PR_RAW_SLOTS * raw_bytes : 0) + 1024;
}

// 2x2/2 max-pool of thresholded bits: out word = OR of the window's words for
// ge channels, AND for le channels (max(v) >= t <=> OR(v_i >= t); max(v) <= t
// <=> AND(v_i <= t)).  One thread per pooled site (all its words; 16-byte
// accesses when a line is 4 words).
__global__ void __launch_bounds__(256) k_pool_bits(const uint32_t* __restrict__ in, int64_t n_img, int h, int w,
                                                   int64_t ldo32, const uint8_t* __restrict__ ge, int c,
                                                   uint32_t* __restrict__ out) {
  pdl_entry();
  __shared__ uint32_t sgm[64];  // ge masks, one word per 32 channels (ldo32 <= 64)
  for (int base = 0; base < (int)ldo32 * 32; base += 256) {
    const int ch = base + (int)threadIdx.x;
    const uint32_t m = __ballot_sync(0xffffffffu, ch < c && __ldg(ge + (ch < c ? ch : 0)) != 0);
    if ((threadIdx.x & 31) == 0 && (ch >> 5) < 64) sgm[ch >> 5] = m;
  }
  __syncthreads();
  const int64_t site = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int hp = h / 2, wp = w / 2;
  if (site >= n_img * hp * wp) return;
  const int64_t n = site / (hp * wp);
  const int rem = (int)(site - n * hp * wp);
  const int py = rem / wp, px = rem - py * wp;
  const int64_t s00 = (n * h + 2 * py) * w + 2 * px;
  const uint32_t* p0 = in + s00 * ldo32;
  const uint32_t* p1 = in + (s00 + w) * ldo32;
  uint32_t* o = out + site * ldo32;
  if (ldo32 == 4) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p0)), b = __ldg(reinterpret_cast<const uint4*>(p0 + 4));
    const uint4 c2 = __ldg(reinterpret_cast<const uint4*>(p1)), d = __ldg(reinterpret_cast<const uint4*>(p1 + 4));
    auto f = [&](uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t gm) {
      return ((x0 | x1 | x2 | x3) & gm) | ((x0 & x1 & x2 & x3) & ~gm);
    };
    *reinterpret_cast<uint4*>(o) = make_uint4(f(a.x, b.x, c2.x, d.x, sgm[0]), f(a.y, b.y, c2.y, d.y, sgm[1]),
                                              f(a.z, b.z, c2.z, d.z, sgm[2]), f(a.w, b.w, c2.w, d.w, sgm[3]));
    return;
  }
  for (int wd = 0; wd < (int)ldo32; ++wd) {
    const uint32_t gm = sgm[wd];
    const uint32_t a = __ldg(p0 + wd), b = __ldg(p0 + ldo32 + wd), c2 = __ldg(p1 + wd), d = __ldg(p1 + ldo32 + wd);
    o[wd] = ((a | b | c2 | d) & gm) | ((a & b & c2 & d) & ~gm);
  }
}

}  // namespace tc
}  // namespace b2
