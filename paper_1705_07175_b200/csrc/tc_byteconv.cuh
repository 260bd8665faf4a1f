// Fused first layer on the int8 tensor cores: byte batch-norm of the raw
// image -> binary convolution -> batch-norm threshold + sign + repack, ONE
// kernel (network.py:128-138 _PackedByteBN, the bit im2col of
// _kernels.py:170-199, layers.py:255-266 conv_forward, _kernels.py:243-267
// threshold_sign_pack).
//
// Row-aligned tiles (as the ALIGN padded-row kernel): a tile is 128
// consecutive output pixels of one image, 128 / W whole rows.  Per tile:
//
//   * producer warps read the tile's input rows (+- pad rows) of u8 pixels,
//     threshold every channel against the byte-BN thresholds into a code of
//     c bits per pixel (shared memory), then assemble each output pixel's
//     window — K = kh kw c bits, (dy, dx, c) order, c fastest, cells in the
//     padding ring marked invalid — and widen it to int8 (+1 / -1, 0 for
//     invalid cells) in one 32-byte A row: one K=32 MMA per tile;
//   * element K of every A row is the constant +1 and element K of filter
//     f's B row holds -t_f (ge) — the filter's other weights negated and +t_f
//     for le filters — so the tensor core returns d = dot - t (ge) or t - dot
//     (le), exact in int32, and the output bit is simply d >= 0: the
//     epilogue extracts sign bits (one funnel shift per element, no
//     threshold table).  Thresholds are clamped to +-(K + 1) (exact, see
//     include/bitnn_b200.h), so |t| <= 32 fits the int8 operand;
//   * the B tile (weights + folded thresholds) is built once per CTA in
//     shared memory from the b2_expand_i8 weights and the thresholds;
//   * four TMEM accumulators (128 columns each) decouple the MMA from the
//     epilogue, whose cost — draining 128 fp32/int32 columns of TMEM per
//     output pixel — bounds the layer.
//
// Operands use the no-swizzle K-major layout: a stage is [2 K planes of 16
// bytes][rows]; LBO = plane stride, SBO = 128 B (8 rows).
#pragma once
#include "tc_padrow.cuh"

namespace b2 {
namespace tc {

struct ByteConvArgs {
  const uint8_t* x;  // (N, H, W, c) u8 image
  int N, H, W, c, kh, kw, pad;
  int64_t HW;
  uint32_t tpi;                 // 128-pixel tiles per image (HW / 128)
  int wshift;                   // log2 W
  int K;                        // kh * kw * c (<= 31): element K carries the threshold
  const int32_t* th_in;         // byte batch-norm thresholds (c), int32 clamped
  const uint8_t* ge_in;
  const int8_t* w;              // b2_expand_i8 rows (K permuted within 32-groups), row pitch wpitch bytes
  int64_t wpitch;
  int F;                        // filters (<= BN)
  const int32_t* thresh;        // output thresholds (F), clamped to +-(K + 1)
  const uint8_t* ge;
  uint32_t* out_bits;           // (N*H*W, ldo32) words
  int64_t ldo32;
};

#ifndef B2_BC_GROUPS  // producer groups (2 -> 3 -> 4: conv1 1.70 -> 1.50 -> 1.16 ms with the later epilogue changes; 896 threads)
#define B2_BC_GROUPS 4
#endif
#ifndef B2_BC_ONE_POLLER
#define B2_BC_ONE_POLLER 0
#endif
#ifndef B2_BC_CHAINS
#define B2_BC_CHAINS 1
#endif
constexpr int BC_GROUPS = B2_BC_GROUPS;
#ifndef B2_BC_PACK16  // epilogue: 16-bit packed TMEM loads + PRMT sign gathering (filters permuted to match)
#define B2_BC_PACK16 1
#endif
// 32 accumulator columns as 16 registers of two int16 halves (column 2j in the
// low half of register j) — the int32 accumulators here are |d| <= 2 (K + 1)
__device__ __forceinline__ void tmem_ld16x2(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
// sign bits of 32 packed columns: PRMT gathers the high bytes of four
// columns (4i .. 4i + 3) into q_i (signs at bits 7, 15, 23, 31), and
// (q_i >> (7 - i)) & (0x01010101 << i) puts column 4i + j at bit 8j + i.
// The B tile's rows are permuted to match (bc_col_filter), so bit f of the
// word is filter f.
__device__ __forceinline__ uint32_t sign_word16(const uint32_t (&v)[16]) {
  uint32_t w = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t q = __byte_perm(v[2 * i], v[2 * i + 1], 0x7531);
    w |= (q >> (7 - i)) & (0x01010101u << i);
  }
  return w;
}
__host__ __device__ constexpr int bc_col_filter(int col) {  // accumulator column -> filter within its 32-chunk
  return (col & ~31) | (8 * (col & 3) + ((col & 31) >> 2));
}  // producer groups working on alternate tiles (independent barriers and bands)
constexpr int BC_NPW = 4 * BC_GROUPS;  // producer warps: per group, one output row per thread
#ifndef B2_BC_STAGES
#define B2_BC_STAGES 8
#endif
constexpr int BC_STAGES = B2_BC_STAGES;  // A stages (4 KB each)
constexpr int BC_NEPI = 8;    // epilogue warps (two per TMEM lane quarter)
#ifndef B2_BC_RAW
#define B2_BC_RAW 3
#endif
constexpr int BC_RAW = B2_BC_RAW;  // raw byte bands in flight per group (TMA, BC_RAW - 1 tiles ahead of the producers)
constexpr int BC_RAW_BYTES = 4096;  // per raw band: (128 / W + 2 pad) rows x W c bytes

template <int BN>
constexpr int bc_acc() {
  return 512 / BN;  // 4 x 128 or 2 x 256 accumulator columns
}
template <int BN>
constexpr int bc_smem_bytes() {
  return BC_STAGES * BM * 32 + BN * 32 + BC_GROUPS * (2 * 4096 + BC_RAW * BC_RAW_BYTES) +  // A ring, B, code + raw bands
         8 * (2 * BC_STAGES + 2 * bc_acc<BN>() + BC_GROUPS * BC_RAW) + 16 + 1024;
}

// KH > 0: compile-time square window (the window gather fully unrolled)
template <int BN, int KH, int C = 0>
__global__ void __launch_bounds__(32 * (4 + BC_NPW + BC_NEPI), 1)
    k_byteconv(const __grid_constant__ CUtensorMap xmap, const ByteConvArgs g) {
  static_assert(C == 0 || KH == 3, "compile-time channels only on the 3x3 path");
  constexpr int ACC = bc_acc<BN>();
  constexpr int EPI0 = 4 + BC_NPW;
  constexpr uint32_t IDESC = idesc_i8(BN, false);
  constexpr int A_BYTES = BM * 32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sa = smem;                                  // BC_STAGES x [2][128][16]
  uint8_t* sbw = sa + BC_STAGES * A_BYTES;             // [2][BN][16]
  uint8_t* scode = sbw + BN * 32;                      // [group][2][1024] pixel codes (u8) / row triples (u32)
  uint8_t* sraw = scode + BC_GROUPS * 2 * 4096;        // [group][BC_RAW][BC_RAW_BYTES] raw image rows (TMA)
  uint64_t* full = reinterpret_cast<uint64_t*>(sraw + BC_GROUPS * BC_RAW * BC_RAW_BYTES);
  uint64_t* empty = full + BC_STAGES;
  uint64_t* tfull = empty + BC_STAGES;
  uint64_t* tempty = tfull + ACC;
  uint64_t* rfull = tempty + ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + BC_GROUPS * BC_RAW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = (int64_t)g.N * g.HW / BM;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < BC_STAGES; ++s) {
      mbar_init(&full[s], BC_NPW / BC_GROUPS);  // the warps of the group that fills stage s
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], BC_NEPI);
    }
    for (int r = 0; r < BC_GROUPS * BC_RAW; ++r) mbar_init(&rfull[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_entry();
  // B tile: filter f's 32 K bytes (permuted like the A rows), le filters
  // negated, the folded threshold at element K; rows past F hold only a -1
  // there (d = -1: their padding bits come out 0, as the layout requires)
  const int kpos = perm_pos(g.K);
  for (int i = threadIdx.x; i < BN * 32; i += blockDim.x) {
    const int col = i >> 5, pos = i & 31;
    // the filter whose dot lands in accumulator column col (permuted for the
    // packed-16-bit epilogue, which the 128-column tiles use)
    const int f = (B2_BC_PACK16 && BN / 32 / (BC_NEPI / 4) <= 2) ? bc_col_filter(col) : col;
    int8_t v = (pos == kpos) ? (int8_t)-1 : (int8_t)0;
    if (f < g.F) {
      const bool ge = __ldg(g.ge + f) != 0;
      if (pos == kpos) {
        // clamping to +-(K + 1) leaves every comparison with |dot| <= K unchanged
        const int32_t t = max(-(g.K + 1), min(g.K + 1, __ldg(g.thresh + f)));
        v = (int8_t)(ge ? -t : t);
      } else {
        const int8_t wv = __ldg(g.w + f * g.wpitch + pos);
        v = ge ? wv : (int8_t)-wv;
      }
    }
    // [plane = pos / 16][row col][16 B]
    sbw[(pos >> 4) * (BN * 16) + col * 16 + (pos & 15)] = (uint8_t)v;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // (the whole warp runs the loop on warp-uniform operands, one elected
    // lane issues: a lone lane-0 issuer spent ~525 cycles per tile around
    // its single MMA — the MMA thread had become this kernel's limit)
    {
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint64_t bdesc = noswz_desc(smem_u32(sbw), BN * 16);
      const uint64_t a0 = noswz_desc(smem_u32(sa), BM * 16);
      const uint32_t a_lo = (uint32_t)a0, a_hi = (uint32_t)(a0 >> 32);
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
#ifdef B2_TC_TIMING
      long long c_acc = 0, c_full = 0, c_t0 = clock64(), c_x;
#endif
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
#ifdef B2_TC_TIMING
        c_x = clock64();
#endif
        mbar_wait(&tempty[acc], aph ^ 1);
#ifdef B2_TC_TIMING
        c_acc += clock64() - c_x, c_x = clock64();
#endif
        mbar_wait(&full[s], ph);
#ifdef B2_TC_TIMING
        c_full += clock64() - c_x;
#endif
        tc_fence_after();
        if (pr_elect<true>()) {
          tc_mma_i8_ss(tm + acc * BN, ((uint64_t)a_hi << 32) | (a_lo + (uint32_t)((s * A_BYTES) >> 4)), bdesc, IDESC, 0u);
          tc_commit(&empty[s]);
          tc_commit(&tfull[acc]);
        }
        if (++s == BC_STAGES) s = 0, ph ^= 1;
        if (++acc == ACC) acc = 0, aph ^= 1;
      }
#ifdef B2_TC_TIMING
      if (blockIdx.x < 2 && lane == 0)
        printf("byteconv cta %d: total %lld  wait acc %lld  wait full %lld  tiles %lld\n", blockIdx.x, clock64() - c_t0,
               c_acc, c_full, (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
#endif
    }
  } else if (warp >= 4 && warp < EPI0) {
    // ------------------------------------------------ producers
    // Raw bytes of a tile's input rows (image rows y0 - pad .. y0 + 128/W - 1
    // + pad, W c bytes each) arrive by TMA two tiles ahead (rows outside
    // the tensor are zero-filled, rows of a neighbouring image are masked
    // below); each thread thresholds its band pixels into codes, the group
    // syncs, and each thread gathers its output pixel's window.  Two groups
    // of four warps take alternate tiles (this CTA's tiles 2j + grp), so one
    // group's barrier and load latencies overlap the other's work.
    const int grp = (warp - 4) >> 2;
    const int pt = threadIdx.x - 4 * 32 - grp * 128;  // 0 .. 127: output row of the tile
    const int wmask = (1 << g.wshift) - 1;
    const int trows = BM >> g.wshift;                 // image rows per tile
    const int brows = trows + 2 * g.pad;              // band rows
    const int bpix = brows << g.wshift;               // band pixels (<= 1024)
    const int rowb = g.W * g.c;                       // bytes per image row
    uint8_t* graw = sraw + grp * BC_RAW * BC_RAW_BYTES;
    uint64_t* grfull = rfull + grp * BC_RAW;
    int32_t tin[3];
    bool gin[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      tin[ch] = ch < g.c ? __ldg(g.th_in + ch) : 0;
      gin[ch] = ch < g.c ? __ldg(g.ge_in + ch) != 0 : true;
    }
    int32_t tq[3];  // compile-time-channel path: t' and the ge mask (see below)
    uint32_t gq = 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      tq[ch] = gin[ch] ? tin[ch] : tin[ch] + 1;
      gq |= (gin[ch] ? 1u : 0u) << ch;
    }
    const int64_t gstep = (int64_t)BC_GROUPS * gridDim.x;  // this group's tile stride
    auto issue = [&](int64_t t, int slot) {  // one thread: TMA of tile t's band rows
      if (t >= tiles) return;
      fence_async_smem();  // the group's reads of this slot (ordered by its barrier) precede the TMA write
      const uint32_t n = (uint32_t)t / g.tpi;  // 32-bit: tiles < 2^31 / 128
      const int y0 = (int)(((uint32_t)t - n * g.tpi) * BM) >> g.wshift;
      mbar_expect_tx(&grfull[slot], (uint32_t)(brows * rowb));
      tma_load_2d(graw + slot * BC_RAW_BYTES, &xmap, &grfull[slot], 0, (int)(n * g.H) + y0 - g.pad);
    };
    const int64_t t0 = blockIdx.x + (int64_t)grp * gridDim.x;
    if (pt == 0)
      for (int r = 0; r + 1 < BC_RAW; ++r) issue(t0 + r * gstep, r);
    int rs = 0;
    uint32_t rph = 0;
    const uint32_t cmask = (1u << g.c) - 1u;
    const int oy = pt >> g.wshift, ox = pt & wmask;  // this thread's output pixel in the tile
    const int kwc = KH > 0 ? KH : g.kw, khc = KH > 0 ? KH : g.kh;
    int cur = 0;
    int64_t i = grp;  // index of tile t among this CTA's tiles: A stage i % BC_STAGES
    for (int64_t t = t0; t < tiles; t += gstep, cur ^= 1, i += BC_GROUPS) {
      if (pt == 0) issue(t + (BC_RAW - 1) * gstep, rs == 0 ? BC_RAW - 1 : rs - 1);  // the slot this group's previous tile used
      const uint32_t n = (uint32_t)t / g.tpi;
      const int y0 = (int)(((uint32_t)t - n * g.tpi) * BM) >> g.wshift;
      mbar_wait(&grfull[rs], rph);
      const uint8_t* raw = graw + rs * BC_RAW_BYTES;
      uint32_t bits = 0, valid = 0;
      if constexpr (KH == 3) {
        // 3x3 (W <= 32, so an image row lies within one warp): every band
        // pixel codes itself and takes its row neighbours' codes by shuffle,
        // storing the ROW TRIPLE (x-1, x, x+1 codes in bits 0..3c-1, their
        // validity in bits 16..) — the window is then three shared loads
        uint32_t* trip = reinterpret_cast<uint32_t*>(scode + (grp * 2 + cur) * 4096);
        for (int b0 = 0; b0 < bpix; b0 += 128) {  // uniform trip count: every lane takes part in the shuffles
          const int b = b0 + pt;
          const int y = y0 - g.pad + (b >> g.wshift);
          const int x = b & wmask;
          uint32_t code = 0, vm = 0;
          if (b < bpix && (unsigned)y < (unsigned)g.H) {
            const int cc = C > 0 ? C : g.c;
            const uint8_t* px = raw + (b >> g.wshift) * rowb + x * cc;
            if constexpr (C > 0) {
              // bit = v >= t (ge) or v <= t = v < t + 1 (le): the sign of
              // v - t' for t' = t (ge) / t + 1 (le), flipped for ge channels
#pragma unroll
              for (int ch = 0; ch < C; ++ch) code |= ((uint32_t)((int32_t)px[ch] - tq[ch]) >> 31) << ch;
              code ^= gq;
            } else {
#pragma unroll
              for (int ch = 0; ch < 3; ++ch)
                if (ch < g.c) code |= (thr_bit((int32_t)px[ch], tin[ch], gin[ch]) ? 1u : 0u) << ch;
            }
            vm = cmask;
          }
          uint32_t cl = __shfl_up_sync(0xffffffffu, code | (vm << 16), 1);
          uint32_t cr = __shfl_down_sync(0xffffffffu, code | (vm << 16), 1);
          if (x == 0) cl = 0;
          if (x == wmask) cr = 0;
          const uint32_t me = code | (vm << 16);
          if (b < bpix) trip[b] = cl | (me << g.c) | (cr << (2 * g.c));
        }
        asm volatile("bar.sync %0, %1;" ::"r"(2 + grp), "n"(128) : "memory");
        if (++rs == BC_RAW) rs = 0, rph ^= 1;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const uint32_t t3 = trip[((oy + dy) << g.wshift) + ox];
          bits |= (t3 & 0xFFFFu) << (dy * 3 * g.c);
          valid |= (t3 >> 16) << (dy * 3 * g.c);
        }
      } else {
      // codes of the band: bit ch = byte-BN bit of channel ch; 0x80 = outside the image
      uint8_t* codes = scode + (grp * 2 + cur) * 4096;
      for (int b = pt; b < bpix; b += 128) {
        const int y = y0 - g.pad + (b >> g.wshift);
        uint32_t code = 0x80u;
        if ((unsigned)y < (unsigned)g.H) {
          const uint8_t* px = raw + (b >> g.wshift) * rowb + (b & wmask) * g.c;
          code = 0;
#pragma unroll
          for (int ch = 0; ch < 3; ++ch)
            if (ch < g.c) code |= (thr_bit((int32_t)px[ch], tin[ch], gin[ch]) ? 1u : 0u) << ch;
        }
        codes[b] = (uint8_t)code;
      }
      // codes ready, raw slot rs consumed (named barrier 2 + group, 128 threads)
      asm volatile("bar.sync %0, %1;" ::"r"(2 + grp), "n"(128) : "memory");
      if (++rs == BC_RAW) rs = 0, rph ^= 1;
      // window bits of this thread's output pixel
      for (int dy = 0; dy < khc; ++dy) {
        for (int dx = 0; dx < kwc; ++dx) {
          const int x = ox + dx - g.pad;
          const int sh = (dy * kwc + dx) * g.c;
          if ((unsigned)x < (unsigned)(wmask + 1)) {
            const uint32_t code = codes[((oy + dy) << g.wshift) + x];
            if (!(code & 0x80u)) {
              bits |= code << sh;
              valid |= cmask << sh;
            }
          }
        }
      }
      }
      bits |= 1u << g.K;  // the constant +1 that carries the threshold
      valid |= 1u << g.K;
      uint32_t o[8];
      widen32m(bits, valid, o);
      const int s = (int)(i % BC_STAGES);
      const uint32_t ph = (uint32_t)(i / BC_STAGES) & 1u;
      mbar_wait_suspend(&empty[s], ph ^ 1);
      uint8_t* st = sa + s * A_BYTES + pt * 16;
      *reinterpret_cast<uint4*>(st) = make_uint4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<uint4*>(st + BM * 16) = make_uint4(o[4], o[5], o[6], o[7]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  } else if (warp >= EPI0) {
    // ------------------------------------------------ epilogue: sign bits of d = +-(dot - t)
    constexpr int ECH = BN / 32 / (BC_NEPI / 4);  // 32-column chunks per warp
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int c0 = ((warp - EPI0) >> 2) * ECH;
    int acc = 0;
    uint32_t aph = 0;
    // this thread's output row of its first tile; rows advance by the grid
    uint32_t* orow = g.out_bits + ((int64_t)blockIdx.x * BM + r) * g.ldo32 + c0;
    const int64_t ostep = (int64_t)gridDim.x * BM * g.ldo32;
    const bool full2 = c0 + 2 <= g.ldo32, one = c0 < g.ldo32;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, orow += ostep) {
#if B2_BC_ONE_POLLER
      if (warp == EPI0) mbar_wait(&tfull[acc], aph);  // one warp polls, the others block in hardware
      epi_bar<BC_NEPI>();
#else
      mbar_wait(&tfull[acc], aph);
#endif
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c0 * 32;
      uint32_t words[ECH];
      if constexpr (ECH <= 2 && B2_BC_PACK16) {
        uint32_t v[ECH][16];
#pragma unroll
        for (int c = 0; c < ECH; ++c) tmem_ld16x2(ta + c * 32, v[c]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
#pragma unroll
        for (int c = 0; c < ECH; ++c) words[c] = ~sign_word16(v[c]);  // bit = d >= 0
      } else if constexpr (ECH <= 2) {
        // both chunks' loads in flight, one wait, then the accumulator is free
        uint32_t v[ECH][32];
#pragma unroll
        for (int c = 0; c < ECH; ++c) tmem_ld32(ta + c * 32, v[c]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
#if B2_BC_CHAINS == 4
#pragma unroll
        for (int c = 0; c < ECH; ++c) words[c] = ~sign_word(v[c]);
#else
#pragma unroll
        for (int c = 0; c < ECH; ++c) {
          uint32_t sg = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) sg = __funnelshift_l(v[c][j], sg, 1);  // sign bits, column 0 at the MSB
          words[c] = ~__brev(sg);
        }
#endif
      } else {
        uint32_t va[32], vb[32];
        tmem_ld32(ta, va);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < ECH; ++c) {
          uint32_t(&v)[32] = (c & 1) ? vb : va;
          uint32_t(&vn)[32] = (c & 1) ? va : vb;
          if (c + 1 < ECH) tmem_ld32(ta + (c + 1) * 32, vn);
          uint32_t sg = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) sg = __funnelshift_l(v[j], sg, 1);
          words[c] = ~__brev(sg);
          if (c + 1 < ECH) tmem_wait_ld();
          if (c + 2 == ECH) {  // every chunk is in registers: return the accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
          }
        }
      }
      uint32_t* o = orow;
      if constexpr (ECH == 2) {
        if (full2) {
          *reinterpret_cast<uint2*>(o) = make_uint2(words[0], words[1]);
        } else if (one) {
          o[0] = words[0];
        }
      } else {
#pragma unroll
        for (int c = 0; c < ECH; ++c)
          if (c0 + c < g.ldo32) o[c] = words[c];
      }
      if (++acc == ACC) acc = 0, aph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tc
}  // namespace b2
