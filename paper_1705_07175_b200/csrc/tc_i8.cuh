// Binary GEMM on the 5th-generation tensor cores (tcgen05 kind::i8, sm_100a).
//
// The XNOR-popcount dot product of the reference
//     dot = K - 2 * popc(a XOR b)                     (_kernels.py:85-106)
// is the integer inner product of the +/-1 vectors the bits encode, so the
// GEMM runs exactly on the int8 tensor pipe once each bit is widened to a
// signed byte (+1 -> 0x01, -1 -> 0xFF) and every element that lies OUTSIDE
// the operand (conv padding sites, K beyond the line) is the byte 0:
//
//   * activations stay bit-packed in HBM (the reference's layout, 1 bit per
//     element); producer warps gather one 128-bit K block per row (implicit
//     bit-im2col for convolutions), widen it in registers and store the 128
//     bytes straight into TENSOR MEMORY with tcgen05.st — the MMA reads A
//     from TMEM, so the widened operand never touches shared memory;
//   * weights are widened once at load (b2_expand_i8) to int8 rows padded
//     to a multiple of 128 with zeros and streamed by TMA (128B swizzle)
//     into a shared-memory ring;
//   * one thread issues tcgen05.mma (M=128, N=BN, K=32 per instruction)
//     into a double-buffered int32 accumulator in TMEM;
//   * epilogue warps tcgen05.ld the accumulator (thread = output row) and
//     apply the reference's stage chain in registers: int32 store, or
//     batchnorm threshold + sign + repack into channel-fastest words, or
//     2x2 max-pool + threshold + repack (rows ordered pool-window-major so
//     the four rows of a window are four adjacent lanes).
//
// Zero bytes for padding make the correction map of the reference
// (layers.py:224-252, added in network.py:193-198) unnecessary: the
// reference's "pad as -1 then add correction" IS the zero-padded product.
//
// Warp roles (512 threads, one persistent CTA per SM, 512 TMEM columns):
//   warp 0      TMA producer for B (one lane)
//   warp 1      MMA issuer (one lane)
//   warp 2      TMEM allocator
//   warps 4-11  A producers (warp%4 = TMEM lane quarter = row quarter;
//               warps 4-7 widen K bits 0-63 of a block, 8-11 bits 64-127)
//   warps 12-15 epilogue     (same lane-quarter rule)
#pragma once
#include <cuda.h>

#include <cstdio>

#include "common.cuh"

namespace b2 {
namespace tc {

constexpr int BM = 128;                 // tile rows = TMEM lanes
constexpr int BK = 128;                 // int8 K of one 128-byte swizzle atom (a TMA box row)
constexpr int KPAD = 512;               // weight rows are padded to a multiple of the widest stage
#ifndef B2_AT_STAGES  // TMEM-A-ring kernels: K stages in flight (0 = as many as fit)
#define B2_AT_STAGES 0
#endif
#ifndef B2_AT_EAGER  // TMEM-A-ring producers: publish each stage right after its store drains (1) or a stage later (0)
#define B2_AT_EAGER 0
#endif
#ifndef B2_PF
#define B2_PF 3  // 3: conv4-6 5-8 % faster than 4 (6: slower; 1-2: between)
#endif
constexpr int PF = B2_PF;                // A-producer prefetch depth (K blocks)

// A operand sources: packed rows; implicit bit-im2col of NHWC-bits
// activations; raw u8 rows; masked window rows of the byte-input first conv
// A_BYTES_TMA: u8 rows loaded by TMA into shared memory (no producer warps;
// the int8 MMA reads A from shared memory)
enum AMode { A_ROWS = 0, A_CONV = 1, A_BYTES = 2, A_BYTECONV = 3, A_BYTES_TMA = 4 };
enum EMode { E_I32 = 0, E_PACK = 1, E_POOLPACK = 2, E_AFFINE = 3 };

struct Args {
  // ---- A operand
  const uint32_t* a;  // packed rows / NHWC-bits activations / bytes (as words)
  int64_t lda;        // A_ROWS/A_BYTES: uint32 words per row
  int awords;         // A_ROWS/A_BYTECONV: valid uint32 words per row (ceil(K/32)); A_BYTES: valid words
  // conv geometry (A_CONV: spw = C/32 words per site; A_BYTECONV: c = channels)
  int H, W, spw, sstride, kh, kw, stride, pad, Ho, Wo, c;
  uint64_t spw_magic, kw_magic;  // ceil(2^32 / spw), ceil(2^32 / kw): exact division of small operands
  // ---- problem
  int64_t M;
  int N;
  int nkb;    // K stages (BKS elements each)
  int klast;  // K=32 MMAs carrying data in the last stage (1..BKS/32)
  int resb;   // the whole B tile (all K stages) stays resident in shared memory:
              // loaded once per CTA (one N tile, nkb stages fit the ring space)
  int ksplit; // split-K kernels: K splits per tile = cluster size (2/4/8)
  // ---- epilogue
  int32_t* out_i32;
  int64_t ldo;
  uint32_t* out_bits;
  int64_t ldo32;
  const int32_t* thresh;
  const uint8_t* ge;
  // E_AFFINE: final float64 batch-norm of the int32 accumulators
  const double* mean;
  const double* scale;
  const double* beta;
  double* out_f64;  // (M, N), leading dimension ldo
  // fp4 packed-output kernels: > 0 = K of the layer, thresholds folded into
  // one more MMA per tile (N columns <= KB_COLS, resident bias block); 0 = table
  int kbias;
};
constexpr int KB_COLS = 512;  // bias-fold column limit (its block reuses the threshold table's 16 KB)

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// 32-bit shared-window address forms (hot loops: no generic -> shared conversion per use)
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_u(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void sts128_u(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// Wait for roles that are not on the MMA's critical path: the thread is
// suspended in hardware until the phase completes (or the hint expires)
// instead of polling, so it does not take issue slots from the MMA thread
// and the producers sharing its SM sub-partition.
__device__ __forceinline__ void mbar_wait_suspend(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}

#ifndef B2_EARLY_RELEASE  // epilogue returns the accumulator once the last TMEM chunk is loaded
#define B2_EARLY_RELEASE 1
#endif
#ifndef B2_TMEM_STAGE  // single 256-column fp4 accumulator: stage half the drain in spare TMEM columns
#define B2_TMEM_STAGE 1
#endif
#ifndef B2_SUSPEND  // 1: TMA, producer and epilogue waits suspend in hardware (the MMA thread polls)
#define B2_SUSPEND 0
#endif
__device__ __forceinline__ void mbar_wait_nc(uint64_t* bar, uint32_t parity) {
  if constexpr (B2_SUSPEND)
    mbar_wait_suspend(bar, parity);
  else
    mbar_wait(bar, parity);
}

// Same wait for roles that idle for long stretches (epilogue, TMA issue):
// back off so their polling does not steal issue slots from the producers.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t done;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}

// TMA into the same offset of every CTA in `mask` (cluster), completing on each one's barrier
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank_u() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Pull [p, p + bytes) into L2 ahead of the producers' gathers (bytes % 16 == 0).
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
#ifndef B2_H2  // half-ordered MMA issue with per-half accumulator barriers (see k_tc_gemm H2)
#define B2_H2 0  // measured slower (conv4 3.18-3.34 vs 3.07 ms with blocks of 1-3 stages): off
#endif
#ifndef B2_H2_R  // K stages per half-ordered block
#define B2_H2_R 3
#endif
#ifndef B2_KB_DRAIN2  // bias-folded single-accumulator drain: two loads, words in between (no spare staging)
#define B2_KB_DRAIN2 1
#endif
#ifndef B2_EPI_ONE_POLLER  // k_tc_gemm epilogue: one warp polls the accumulator barrier, the rest wait on bar.sync
#define B2_EPI_ONE_POLLER 0  // with the warp-issued TMEM-ring kernels all-warp polling measured 1-3 % faster (conv6 3.02 -> 2.93 ms)
#endif
#ifndef B2_CONV_FAST  // lean fp4 conv producer (ConvCursor); 0 = the general ACursor
#define B2_CONV_FAST 0  // measured slower than the general cursor (conv4 3.92 vs 3.62 ms) for reasons not yet understood
#endif
#ifndef B2_TC_WI_F4  // fp4 shared-memory kernels: warp-wide uniform MMA issue too
#define B2_TC_WI_F4 1
#endif
#ifndef B2_TC_WARP_ISSUE
#define B2_TC_WARP_ISSUE 0  // measured slower on the im2col kernel (conv4 3.65 -> 4.26 ms)
#endif
// WI: one lane of the converged issuing warp (the lowest active) issues;
// otherwise the issuing code runs on lane 0 alone
template <bool WI>
__device__ __forceinline__ bool pr_elect() {
  if constexpr (WI) {
    uint32_t e;
    asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p;}" : "=r"(e));
    return e != 0;
  } else {
    return true;
  }
}

// kind::mxf4 with A from TMEM (TS form)
__device__ __forceinline__ void tc_mma_f4_ts_g(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t sfa_tmem, uint32_t sfb_tmem, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem)
      : "memory");
}
// MMA completion -> arrive on `bar` in every CTA of `mask`
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// ---- thread-block cluster (split-K reduction over distributed shared memory)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t saddr, uint32_t rank) {  // my smem address -> rank's
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// Work item t of a kernel with ksp K splits per tile: tile t / ksp, K
// stages [kb0, kb1) of split t % ksp (ksp = 1: the whole K walk).
__device__ __forceinline__ void item_krange(const Args& g, int ksp, int64_t t, int& kb0, int& kb1) {
  const int s = (int)(t % ksp);
  kb0 = s * g.nkb / ksp;
  kb1 = (s + 1) * g.nkb / ksp;
}

#define B2_R32(v)                                                                                                   \
  "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),    \
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),   \
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),   \
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define B2_W32(v)                                                                                                   \
  "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),      \
      "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),        \
      "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),       \
      "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])

// 32 consecutive TMEM columns of this thread's lane <- v[0..31]
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      B2_R32(v)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : B2_W32(v)
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// K-major operand, 128-byte swizzle: 8-row atoms of 128 B, atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// instruction descriptor: D s32, A s8|u8, B s8, both K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int n, bool a_unsigned) {
  return (2u << 4) | ((a_unsigned ? 0u : 1u) << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

// 32 bits (elements k..k+31, LSB first) -> 32 signed bytes in 8 words,
// bit 1 -> +1 (0x01), bit 0 -> -1 (0xFF); an invalid (padding) word -> 0.
// K is PERMUTED inside each 32-element group: byte j of output word s holds
// element 8j + s, so each output word is one shift, one mask and one IMAD.
// The weights are widened with the same permutation (k_expand_i8); a dot
// product is invariant under a common permutation of K.
__device__ __forceinline__ void widen32(uint32_t x, bool ok, uint32_t* o) {
  const uint32_t nx = ok ? ~x : 0u;
  const uint32_t c = ok ? 0x01010101u : 0u;
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = ((nx >> q) & 0x01010101u) * 0xFEu + c;
}
__host__ __device__ __forceinline__ int perm_pos(int k) {  // element k of a 32-group -> byte position
  return 4 * (k & 7) + (k >> 3);
}

// Output row -> (image, oy, ox); pool-ordered rows put each 2x2 window in
// four consecutive rows: m = 4*q + 2*cy + cx.
// 32-bit arithmetic: the conv entry points require M < 2^31.
template <bool POOLED>
__device__ __forceinline__ void row_pos(const Args& g, int64_t m, int64_t& img, int& oy, int& ox) {
  const uint32_t mm = (uint32_t)m;
  if constexpr (POOLED) {
    const uint32_t q = mm >> 2;
    const uint32_t cell = mm & 3u;
    const uint32_t hp = (uint32_t)g.Ho >> 1, wp = (uint32_t)g.Wo >> 1;
    const uint32_t im = q / (hp * wp);
    const uint32_t r = q - im * (hp * wp);
    const uint32_t ry = r / wp;
    img = im;
    oy = (int)(2 * ry + (cell >> 1));
    ox = (int)(2 * (r - ry * wp) + (cell & 1));
  } else {
    const uint32_t hw = (uint32_t)g.Ho * (uint32_t)g.Wo;
    const uint32_t im = mm / hw;
    const uint32_t r = mm - im * hw;
    const uint32_t y = r / (uint32_t)g.Wo;
    img = im;
    oy = (int)y;
    ox = (int)(r - y * (uint32_t)g.Wo);
  }
}

// persistent tile loops advance t by the grid size: keep (m tile, n tile)
// incrementally, dividing only when the m index wraps
__device__ __forceinline__ void next_tile(int64_t& mt, int64_t& nt, int64_t step, int64_t mtiles) {
  mt += step;
  if (mt >= mtiles) {
    nt += mt / mtiles;
    mt %= mtiles;
  }
}

// Per-bit-masked variant for the byte-batchnorm first layer: bits whose
// valid bit is 0 (window cells in the padding ring) become the byte 0.
__device__ __forceinline__ void widen32m(uint32_t x, uint32_t valid, uint32_t* o) {
  const uint32_t nx = ~x & valid;
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = ((nx >> q) & 0x01010101u) * 0xFEu + ((valid >> q) & 0x01010101u);
}

// ---- fp4 operands (tcgen05.mma kind::mxf4, e2m1 with unit block scales).
// +1.0 = 0x2, -1.0 = 0xA, 0 = 0x0 are exact in e2m1; products are +/-1 and
// the fp32 accumulator holds the exact integer dot product (|dot| < 2^24).
// 32 bits -> 32 nibbles (4 words, 16 bytes): nibble i of word q holds
// element 4i + q (a common permutation of K within each 32-group, applied to
// the weights too by k_expand_f4): one shift and one LOP3 per word.
// Branch-free: with m = all ones for a valid word (else 0), nibble =
// 0x2 (valid) | 0x8 (valid and bit 0): one LOP3 for ~x & m, then a shift and
// one LOP3 per output word.
__device__ __forceinline__ void widen_f4(uint32_t x, bool ok, uint32_t* o) {
  const uint32_t m = 0u - (uint32_t)ok;
  const uint32_t nx = ~x & m, c2 = m & 0x22222222u;
  o[0] = ((nx << 3) & 0x88888888u) | c2;
  o[1] = ((nx << 2) & 0x88888888u) | c2;
  o[2] = ((nx << 1) & 0x88888888u) | c2;
  o[3] = (nx & 0x88888888u) | c2;
}
__device__ __forceinline__ void widen_f4m(uint32_t x, uint32_t valid, uint32_t* o) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    o[q] = (0xAAAAAAAAu ^ ((x << (3 - q)) & 0x88888888u)) & (((valid >> q) & 0x11111111u) * 0xFu);
}
__host__ __device__ __forceinline__ int perm_pos_f4(int k) {  // element k of a 32-group -> nibble position
  return 8 * (k & 3) + (k >> 2);
}
// instruction descriptor, kind::mxf4: A/B e2m1 (1), both K-major, UE8M0
// scales, M = 128, K = 64 per instruction (cute InstrDescriptorBlockScaled)
__host__ __device__ constexpr uint32_t idesc_f4(int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_f4(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t sfa_tmem, uint32_t sfb_tmem, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {  // generic-proxy smem writes -> tensor-core reads
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Gather cursor of one A-producer thread (one tile row, one half of each
// 128-element K block): walks this CTA's (tile, K block) sequence.
//   A_ROWS / A_CONV / A_BYTECONV: 64 packed bits (uint2) + validity
//   A_BYTES:                      64 raw bytes (4 x uint4)
// DIRECT (conv): every chunk's window cell and word are computed from its
// absolute K word (no incremental cell walk, no branches).
__device__ __forceinline__ uint32_t div_magic(uint32_t n, uint64_t magic) {  // n / d, n < 2^16, d < 2^16
  return (uint32_t)(((uint64_t)n * magic) >> 32);
}
// Lean conv cursor (fp4, packed-bit input, no split-K, <= 32 window cells):
// per tile the row's image site pointer and a bit mask of its in-image
// window cells; per stage 32-bit offset arithmetic only.  The general cursor
// spent ~250 instructions per (row, stage) on 64-bit addressing, per-fetch
// cell decoding and tile bookkeeping (ncu: the producers issued 45 % of the
// im2col kernel's instructions, and the kernel was issue-bound).
template <bool POOLED, int WS, int WPH>
struct ConvCursor {
  int64_t t;
  int kb;
  const uint32_t* rowp;  // site (iy0, ix0) of this row's window (may lie outside the image; read only if valid)
  uint32_t vmask;        // window cells inside the image (0 for rows past M / tiles past the end)
  int cell, within, dx, off;
  __device__ __forceinline__ void tile(const Args& g, int64_t mtiles, int64_t tiles, int r, int half) {
    kb = 0;
    const int64_t m = (t % mtiles) * BM + r;
    const bool mok = t < tiles && m < g.M;
    int64_t img = 0;
    int oy = 0, ox = 0;
    if (mok) row_pos<POOLED>(g, m, img, oy, ox);
    const int iy0 = oy * g.stride - g.pad, ix0 = ox * g.stride - g.pad;
    vmask = 0;
    if (mok)
      for (int dy = 0, c = 0; dy < g.kh; ++dy)
        for (int dx_ = 0; dx_ < g.kw; ++dx_, ++c)
          if ((unsigned)(iy0 + dy) < (unsigned)g.H && (unsigned)(ix0 + dx_) < (unsigned)g.W) vmask |= 1u << c;
    rowp = g.a + ((img * g.H + iy0) * g.W + ix0) * g.sstride;
    const int w = WPH * half;  // this thread's first K word of stage 0
    cell = w / g.spw;
    within = w - cell * g.spw;
    const int dy = cell / g.kw;
    dx = cell - dy * g.kw;
    off = (dy * g.W + dx) * g.sstride;
  }
  __device__ __forceinline__ void start(const Args& g, int64_t t0, int64_t mtiles, int64_t tiles, int r, int half) {
    t = t0;
    tile(g, mtiles, tiles, r, half);
  }
  __device__ __forceinline__ void fetch(uint4& x, bool& ok) const {
    ok = (vmask >> cell) & 1u;
    x = ok ? __ldg(reinterpret_cast<const uint4*>(rowp + off + within)) : make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ void advance(const Args& g, int64_t step, int64_t mtiles, int64_t tiles, int r,
                                          int half) {
    if (++kb == g.nkb) {
      t += step;
      tile(g, mtiles, tiles, r, half);
      return;
    }
    within += WS;
    while (within >= g.spw) {
      within -= g.spw;
      ++cell;
      if (++dx == g.kw)
        dx = 0, off += (g.W - g.kw + 1) * g.sstride;
      else
        off += g.sstride;
    }
  }
};
// 32 bits -> 4 words of e2m1 +-1 nibbles (widen_f4's order) with the sign
// pattern XORed in: 2 instructions per word; c2 = 0xAAAAAAAA for a valid
// word (x = 0 and c2 = 0 give 0 nibbles)
__device__ __forceinline__ void widen_f4x(uint32_t x, uint32_t c2, uint32_t* o) {
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = ((x << (3 - q)) & 0x88888888u) ^ c2;
}

template <int AM, bool POOLED, int WS, int TW, bool DIRECT = false>  // WS = K words per stage, TW = words per producer thread
struct ACursor {
  int64_t t;       // work item of the next fetch (tile t / ksp)
  int64_t mt, nt_; // m (and n) tile of t, kept incrementally when ksp == 1
  int kb, kend;    // K block of the next fetch, end of the item's K range
  bool mok;        // row inside M
  const uint32_t* base;
  int iy0, ix0;    // conv: window origin of this row
  int cell, within, dy, dx;  // conv: window cell and word of this half's next K words
  int64_t img;

  __device__ __forceinline__ void tile_setup(const Args& g, int64_t mtiles, int64_t tiles, int r, int half,
                                             int ksp) {
    item_krange(g, ksp, t, kb, kend);
    const int64_t m = mt * BM + r;
    mok = t < tiles * ksp && m < g.M;
    if constexpr (AM == A_CONV) {
      img = 0;
      int oy = 0, ox = 0;
      if (mok) row_pos<POOLED>(g, m, img, oy, ox);
      iy0 = oy * g.stride - g.pad;
      ix0 = ox * g.stride - g.pad;
      base = g.a + img * (int64_t)g.H * g.W * g.sstride;
      if constexpr (!DIRECT) {
        cell = dy = dx = 0;
        within = TW * half + kb * WS;  // this producer warp's first word of the item's first stage
        while (within >= g.spw) within -= g.spw, step_cell(g);
      }
    } else {
      base = g.a + (mok ? m : 0) * g.lda;
    }
  }
  __device__ __forceinline__ void step_cell(const Args& g) {
    ++cell;
    if (++dx == g.kw) dx = 0, ++dy;
  }
  __device__ __forceinline__ void start(const Args& g, int64_t t0, int64_t mtiles, int64_t tiles, int r, int half,
                                        int ksp) {
    t = t0;
    mt = (t0 / ksp) % mtiles;
    nt_ = 0;
    tile_setup(g, mtiles, tiles, r, half, ksp);
  }
  __device__ __forceinline__ void advance(const Args& g, int64_t step, int64_t mtiles, int64_t tiles, int r,
                                          int half, int ksp) {
    if (++kb == kend) {
      t += step;
      if (ksp == 1)
        next_tile(mt, nt_, step, mtiles);
      else
        mt = (t / ksp) % mtiles;
      tile_setup(g, mtiles, tiles, r, half, ksp);
    } else if constexpr (AM == A_CONV && !DIRECT) {
      within += WS;
      while (within >= g.spw) within -= g.spw, step_cell(g);
    }
  }

  // DIRECT conv: address of K word `wpos` of this row's window (site
  // cell = wpos / spw, word within the site, cell -> (dy, dx)); ok = in bounds
  __device__ __forceinline__ const uint32_t* conv_word(const Args& g, int wpos, bool& ok) const {
    const uint32_t cell = div_magic((uint32_t)wpos, g.spw_magic);
    const int within_ = wpos - (int)cell * g.spw;
    const uint32_t dy_ = div_magic(cell, g.kw_magic);
    const int dx_ = (int)cell - (int)dy_ * g.kw;
    const int iy = iy0 + (int)dy_, ix = ix0 + dx_;
    ok = mok && (int)dy_ < g.kh && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W;
    return base + ((int64_t)iy * g.W + ix) * g.sstride + within_;
  }

  // packed-bit modes: x = WPH words (32 bits each) of K starting at word
  // 4 kb + WPH half, vm = validity (all ones / zero, or per bit for
  // A_BYTECONV).  WPH = 2 (two producer warps per lane quarter) or 4 (one).
  template <int WPH>
  __device__ __forceinline__ void fetch_bits(const Args& g, int half, uint4& x, uint4& vm) {
    x = make_uint4(0, 0, 0, 0);
    vm = make_uint4(0, 0, 0, 0);
    if constexpr (AM == A_ROWS) {
      const int w0 = kb * WS + WPH * half;
      if (mok) {
        vm = make_uint4(~0u, ~0u, ~0u, ~0u);
        const uint32_t* p = base + w0;
        if (WPH == 4 && w0 + 4 <= g.awords && (g.lda & 3) == 0) {
          x = __ldg(reinterpret_cast<const uint4*>(p));
        } else if (WPH == 2 && w0 + 2 <= g.awords && (g.lda & 1) == 0) {
          const uint2 y = __ldg(reinterpret_cast<const uint2*>(p));
          x.x = y.x, x.y = y.y;
        } else {
          if (w0 + 0 < g.awords) x.x = __ldg(p + 0);
          if (w0 + 1 < g.awords) x.y = __ldg(p + 1);
          if (WPH == 4 && w0 + 2 < g.awords) x.z = __ldg(p + 2);
          if (WPH == 4 && w0 + 3 < g.awords) x.w = __ldg(p + 3);
        }
      }
    } else if constexpr (AM == A_CONV && DIRECT) {
      bool ok;
      const uint32_t* p = conv_word(g, kb * WS + WPH * half, ok);
      if (ok) {
        vm = make_uint4(~0u, ~0u, ~0u, ~0u);
        if constexpr (WPH == 4) {
          x = __ldg(reinterpret_cast<const uint4*>(p));
        } else {
          const uint2 y = __ldg(reinterpret_cast<const uint2*>(p));
          x.x = y.x, x.y = y.y;
        }
      }
    } else if constexpr (AM == A_CONV) {
      // WPH consecutive K words of one site (spw % WPH == 0)
      const int iy = iy0 + dy, ix = ix0 + dx;
      if (mok && dy < g.kh && iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) {
        vm = make_uint4(~0u, ~0u, ~0u, ~0u);
        const uint32_t* p = base + ((int64_t)iy * g.W + ix) * g.sstride + within;
        if constexpr (WPH == 4) {
          x = __ldg(reinterpret_cast<const uint4*>(p));
        } else {
          const uint2 y = __ldg(reinterpret_cast<const uint2*>(p));
          x.x = y.x, x.y = y.y;
        }
      }
    } else if constexpr (AM == A_BYTECONV) {
      // masked rows written by k_byte_unroll: awords bit words then awords
      // validity words per row (padding cells of the window -> byte 0)
      const int w0 = kb * WS + WPH * half;
      if (mok) {
        const uint32_t* p = base + w0;
        if (w0 + 0 < g.awords) x.x = __ldg(p + 0), vm.x = __ldg(p + g.awords + 0);
        if (w0 + 1 < g.awords) x.y = __ldg(p + 1), vm.y = __ldg(p + g.awords + 1);
        if (WPH == 4 && w0 + 2 < g.awords) x.z = __ldg(p + 2), vm.z = __ldg(p + g.awords + 2);
        if (WPH == 4 && w0 + 3 < g.awords) x.w = __ldg(p + 3), vm.w = __ldg(p + g.awords + 3);
      }
    }
  }
  // 8 words (two 4-word chunks) per producer thread: 512-element stages.
  // ok[j] = chunk j lies inside the operand (conv: its site is in bounds).
  __device__ __forceinline__ void fetch_bits8(const Args& g, int half, uint4 (&x)[2], bool (&ok)[2]) {
    x[0] = x[1] = make_uint4(0, 0, 0, 0);
    ok[0] = ok[1] = false;
    if constexpr (AM == A_ROWS) {
      const int w0 = kb * WS + 8 * half;
      ok[0] = ok[1] = mok;
      if (mok) {
        const uint32_t* p = base + w0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int w = w0 + 4 * j;
          if (w + 4 <= g.awords && (g.lda & 3) == 0) {
            x[j] = __ldg(reinterpret_cast<const uint4*>(p + 4 * j));
          } else {
            if (w + 0 < g.awords) x[j].x = __ldg(p + 4 * j + 0);
            if (w + 1 < g.awords) x[j].y = __ldg(p + 4 * j + 1);
            if (w + 2 < g.awords) x[j].z = __ldg(p + 4 * j + 2);
            if (w + 3 < g.awords) x[j].w = __ldg(p + 4 * j + 3);
          }
        }
      }
    } else if constexpr (AM == A_CONV && DIRECT) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t* p = conv_word(g, kb * WS + 8 * half + 4 * j, ok[j]);
        if (ok[j]) x[j] = __ldg(reinterpret_cast<const uint4*>(p));
      }
    } else if constexpr (AM == A_CONV) {
      // chunk 0 at the cursor's (cell, within); chunk 1 four words later
      int cw = within, cy = dy, cx = dx;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j) {
          cw += 4;
          while (cw >= g.spw) {
            cw -= g.spw;
            if (++cx == g.kw) cx = 0, ++cy;
          }
        }
        const int iy = iy0 + cy, ix = ix0 + cx;
        ok[j] = mok && cy < g.kh && iy >= 0 && iy < g.H && ix >= 0 && ix < g.W;
        if (ok[j]) x[j] = __ldg(reinterpret_cast<const uint4*>(base + ((int64_t)iy * g.W + ix) * g.sstride + cw));
      }
    }
  }

  // A_BYTES: bytes [128 kb + 64 half, +64) of the row (awords = valid words; WS == 4)
  __device__ __forceinline__ void fetch_bytes(const Args& g, int half, uint4 (&x)[4]) {
    const int w0 = kb * 32 + 16 * half;
    const bool vec = (g.lda & 3) == 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] = make_uint4(0, 0, 0, 0);
      const int w = w0 + 4 * i;
      if (!mok || w >= g.awords) continue;
      if (vec && w + 4 <= g.awords) {
        x[i] = __ldg(reinterpret_cast<const uint4*>(base + w));
      } else {  // row tail or a row pitch that is not 16-byte aligned
        x[i].x = __ldg(base + w);
        if (w + 1 < g.awords) x[i].y = __ldg(base + w + 1);
        if (w + 2 < g.awords) x[i].z = __ldg(base + w + 2);
        if (w + 3 < g.awords) x[i].w = __ldg(base + w + 3);
      }
    }
  }
};

// Pipeline shape per (BN, A mode).  Two independent rings: the shared-memory
// B ring (TMA) and the TMEM A ring (producers); the MMA waits on both.
// TMEM holds ACC_BUFS accumulators of BN columns plus A_STAGES A stages of
// 32 columns (512 columns in all).  The B ring is as deep as shared memory
// allows (192 KB) so TMA runs >= 3 us ahead of the tensor cores.  The
// first conv has one K block per tile, so its accumulator ring is deeper
// (3 x 128) to hide the MMA -> epilogue hand-off, with a 4-stage A ring.
// L2 prefetch of the input rows tile `t` will gather (implicit im2col:
// the NHWC-bits rows oy0*stride-pad .. oy1*stride-pad+kh-1 of the tile's
// images are one contiguous range; packed rows: the tile's A rows).
template <int AM>
__device__ __forceinline__ void prefetch_tile_inputs(const Args& g, int64_t t, int64_t mtiles, int64_t tiles) {
  if (t >= tiles) return;
  const int64_t m0 = (t % mtiles) * BM;
  const int64_t m1 = (m0 + BM < g.M ? m0 + BM : g.M) - 1;
  int64_t lo, hi;  // uint32 word range
  if constexpr (AM == A_CONV) {
    // pool-ordered rows stay within the same output-row band as natural ones
    const int64_t hw = (int64_t)g.Ho * g.Wo;
    const int64_t i0 = m0 / hw, i1 = m1 / hw;
    const int oy0 = (int)((m0 - i0 * hw) / g.Wo), oy1 = (int)((m1 - i1 * hw) / g.Wo);
    int y0 = oy0 * g.stride - g.pad, y1 = oy1 * g.stride - g.pad + g.kh;
    y0 = y0 < 0 ? 0 : y0;
    y1 = y1 > g.H ? g.H : y1;
    lo = (i0 * g.H + y0) * (int64_t)g.W * g.sstride;
    hi = (i1 * g.H + y1) * (int64_t)g.W * g.sstride;
  } else {
    lo = m0 * g.lda;
    hi = (m1 + 1) * g.lda;
  }
  const uint8_t* p = reinterpret_cast<const uint8_t*>(g.a + lo);
  int64_t bytes = (hi - lo) * 4;
  const uintptr_t mis = reinterpret_cast<uintptr_t>(p) & 15;
  p -= mis;
  bytes = (bytes + mis + 15) & ~int64_t(15);
  while (bytes > 0) {
    const uint32_t n = bytes > (1 << 20) ? (1u << 20) : (uint32_t)bytes;
    l2_prefetch(p, n);
    p += n;
    bytes -= n;
  }
}

// K elements per pipeline stage (BKS): 256 for 128-column tiles (8 MMAs of
// 64 cycles between the two ring commits — at 4 per stage the commits and
// the issuing thread's waits cost ~40 % of the tensor pipe), else 128.
#ifndef B2_ACC128
#define B2_ACC128 2  // accumulator buffers of 128-column tiles (experiments: 1 buys a third A stage)
#endif
template <int BN, int AM>
constexpr int acc_bufs() {
  return BN > 128 ? 1 : (AM == A_BYTECONV ? 3 : (B2_ACC128));
}
template <int BN, int AM, int BKS>
constexpr int a_stages() {  // TMEM: accumulators + A ring fill the 512 columns
  return (512 - acc_bufs<BN, AM>() * BN) / (BKS / 4);
}
template <int BN, int BKS>
constexpr int b_stages() {  // 192 KB of shared memory for the B ring
  return (192 * 1024) / (BN * BKS);
}
// fp4 (kind::mxf4): A and B stages both in shared memory, 4 bits per
// element; the ring holds f4_stages() of each in 192 KB.  TMEM holds only
// accumulators (3 x 128 or 1 x 256 columns) and the unit scale factors.
template <int BN, int BKS>
constexpr int at_stages() {  // fp4 with A in TMEM: B stages in 192 KB, A stages in TMEM columns past 288
  constexpr int n = (192 * 1024) / (BN * BKS / 2) < (512 - BN - 32) / (BKS / 8) ? (192 * 1024) / (BN * BKS / 2)
                                                                               : (512 - BN - 32) / (BKS / 8);
  return B2_AT_STAGES > 0 && B2_AT_STAGES < n ? B2_AT_STAGES : n;
}
template <int BN, int BKS>
constexpr int f4_stages() {
  return (192 * 1024) / ((BN + BM) * BKS / 2);
}
template <int BN>
constexpr int f4_acc_bufs() {
  return BN > 128 ? 1 : 3;
}
constexpr int F4_SF_COLS = 16;  // TMEM columns of 0x7F (2^0) scale bytes, after the accumulators

template <int NEPI>
__device__ __forceinline__ void epi_bar() {  // named barrier of the epilogue warps
  asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");
}

constexpr int THR_COLS = 2048;  // resident threshold table (columns)

// Threshold table for columns [n0, n0 + ncols) (ncols % nthr == 0), built
// by the nthr epilogue threads (et = 0 .. nthr-1): ge -> (1, -t), le ->
// (-1, t), column beyond N -> (0, -1) = bit 0; one ge-direction mask word
// per 32 columns (ballot).
template <bool F4 = false>
__device__ __forceinline__ void stage_thresholds(const Args& g, int n0, int ncols, int et, int nthr, int lane,
                                                 int4* sthr, uint32_t* sgm) {
  int* st = reinterpret_cast<int*>(sthr);
  for (int j = et; j < ncols; j += nthr) {
    const int n = n0 + j;
    int mul = 0, add = -1;
    bool ge = true;
    if (n < g.N) {
      const int32_t th = __ldg(g.thresh + n);
      ge = __ldg(g.ge + n) != 0;
      mul = ge ? 1 : -1;
      add = ge ? -th : th;
    }
    if (!sthr) {  // bias fold: the direction masks only
    } else if constexpr (F4) {  // fp32 accumulators: (mul, add) as floats (|add| < 2^24 exact; larger only for sentinels)
      st[2 * j] = __float_as_int((float)mul);
      st[2 * j + 1] = __float_as_int((float)add);
    } else {
      st[2 * j] = mul;
      st[2 * j + 1] = add;
    }
    const uint32_t gmw = __ballot_sync(0xffffffffu, ge);
    if (lane == 0) sgm[j >> 5] = gmw;
  }
}

// K-major, no swizzle: 8-row x 16-byte core matrices, LBO = K-plane stride, SBO = 128
__device__ __forceinline__ uint64_t noswz_desc_k(uint32_t saddr, uint32_t kplane_bytes) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((kplane_bytes >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((128u >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// ---- threshold folded into the GEMM (tc_padrow.cuh BIAS, k_tc_gemm kbias):
// one more K = 64 MMA per tile adds a per-filter integer bias -T' to every
// accumulator, so the epilogue only collects sign bits.  A = a constant +1
// block, B = the filter's 64 bias elements: block 0 (scale 2^5) holds 16 q,
// block 1 (scale 2^0) the rest r, b = 16 q + r.  T' = T (ge: bit = acc >= T,
// sign clear) or T + 1 (le: bit = acc <= T, sign set), clamped to +-(K + 1).
constexpr uint32_t PR_BIAS_SF = 0x7F7F7F84u;  // scale bytes: block 0 2^5, block 1 2^0
// e2m1 magnitudes of a count of half units (<= 11): up to two codes
__device__ __forceinline__ void pr_half_units(int h, int& c0, int& c1) {
  // 0.5 1 1.5 2 3 4 6 -> codes 1..7 = 1 2 3 4 6 8 12 half units
  static constexpr int8_t a[12] = {0, 1, 2, 3, 4, 4, 5, 5, 6, 6, 6, 6};
  static constexpr int8_t b[12] = {0, 0, 0, 0, 0, 1, 0, 1, 0, 1, 2, 3};
  c0 = a[h], c1 = b[h];
}
// 32 e2m1 codes (one scale block) summing to sign * h half units, h <= 30 * 12 + 11
__device__ __forceinline__ uint4 pr_bias_block(int h, bool neg) {
  uint32_t w[4] = {0, 0, 0, 0};
  const uint32_t sg = neg ? 8u : 0u;
  int e = 0;
  for (; h >= 12; h -= 12, ++e) w[e >> 3] |= (7u | sg) << (4 * (e & 7));
  int c0, c1;
  pr_half_units(h, c0, c1);
  if (c0) w[e >> 3] |= ((uint32_t)c0 | sg) << (4 * (e & 7)), ++e;
  if (c1) w[e >> 3] |= ((uint32_t)c1 | sg) << (4 * (e & 7)), ++e;
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// the 32 bytes of filter n's threshold block
__device__ __forceinline__ void pr_bias_bytes(int64_t bias, uint4& blk0, uint4& blk1) {
  const int64_t q = bias / 16, r = bias - 16 * q;  // |r| < 16
  blk0 = pr_bias_block((int)(q < 0 ? -q : q), q < 0);        // q half units of 2^5 = 16 q
  blk1 = pr_bias_block((int)(2 * (r < 0 ? -r : r)), r < 0);  // 2 |r| half units of 2^0 = r
}
// sign word of 32 accumulators: bit j = sign bit of v[j]
__device__ __forceinline__ uint32_t sign_word(const uint32_t (&v)[32]) {
  uint32_t sg = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) sg = __funnelshift_l(v[j], sg, 1);
  return __brev(sg);
}

// bias of filter n for K-element dot products (padding filters: -1 = bit 0 with ge)
__device__ __forceinline__ int64_t filter_bias(const int32_t* thresh, const uint8_t* ge, int n, int nvalid, int64_t k) {
  if (n >= nvalid) return -1;
  const int64_t th = __ldg(thresh + n);
  const int64_t b = __ldg(ge + n) ? -th : -(th + 1);
  return b > k + 1 ? k + 1 : (b < -(k + 1) ? -(k + 1) : b);
}
// Packed sign word of 32 accumulators: bit j = (v[j] * mul_j + add_j >= 0)
// with trow = the columns' (mul, add) pairs (sign bits MSB first, reversed).
// F4: v holds fp32 accumulators and the table float (mul, add); the sign of
// the exact fma is the sign of the integer form.
template <bool F4 = false>
__device__ __forceinline__ uint32_t thr_word(const uint32_t (&v)[32], const int4* trow) {
  uint32_t sg = 0;
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const int4 p = trow[j / 2];
    uint32_t d0, d1;
    if constexpr (F4) {
      d0 = __float_as_uint(fmaf(__uint_as_float(v[j]), __int_as_float(p.x), __int_as_float(p.y)));
      d1 = __float_as_uint(fmaf(__uint_as_float(v[j + 1]), __int_as_float(p.z), __int_as_float(p.w)));
    } else {
      d0 = (uint32_t)((int)v[j] * p.x + p.y);
      d1 = (uint32_t)((int)v[j + 1] * p.z + p.w);
    }
    sg = __funnelshift_l(d0, sg, 1);
    sg = __funnelshift_l(d1, sg, 1);
  }
  return ~__brev(sg);
}
template <bool F4>
__device__ __forceinline__ int acc_int(uint32_t v) {  // accumulator -> exact integer
  if constexpr (F4)
    // |v| < 2^22 (K <= 2^22, the entry points' limit): v + 1.5 * 2^23 holds v
    // in its low mantissa bits — an FADD and an integer subtract on the full-
    // rate pipes instead of the quarter-rate F2I
    return (int)(__float_as_uint(__fadd_rn(__uint_as_float(v), 12582912.0f)) - 0x4B400000u);
  else
    return (int)v;
}
// 2x2 max-pool of thresholded rows held by 4 consecutive lanes: max then
// threshold == OR (ge columns, mask gm) / AND (le) of the four words
__device__ __forceinline__ uint32_t pool_word(uint32_t w, uint32_t gm) {
  uint32_t o = w | __shfl_xor_sync(0xffffffffu, w, 1);
  o |= __shfl_xor_sync(0xffffffffu, o, 2);
  uint32_t a = w & __shfl_xor_sync(0xffffffffu, w, 1);
  a &= __shfl_xor_sync(0xffffffffu, a, 2);
  return (o & gm) | (a & ~gm);
}

// ------------------------------------------------------------------ kernel
template <int NPW, int NEPI>
constexpr int num_threads() {
  return 32 * (4 + NPW + NEPI);
}

// NPW A-producer warps: 8 (two per TMEM lane quarter, 64 K elements each)
// or 4 (one per quarter, the whole 128-element block: per-stage overheads
// amortised over twice the widening, for 128-column tiles).
// NEPI epilogue warps: 4 (one per lane quarter, all columns) or 8 (two per
// quarter, half the columns each: TMEM reads are latency-bound per warp,
// ~42 B/clk each, so a single-buffered 256-column accumulator drains twice
// as fast).
// KB: thresholds folded into one more MMA per tile (Args.kbias = K; packed
// fp4 output, <= KB_COLS columns): a separate instantiation, so the
// threshold-table kernels keep their register allocation
// MC: the two CTAs of a cluster share each weight (B) stage: each loads half
// its rows by TMA multicast into both CTAs' shared memory, and both MMAs'
// commits release the stage in both (conv4-6 stream every B stage once per
// 128-pixel tile; the three layers sat at 10-12 TB/s of L2->SM weight
// traffic, the L2's ceiling).  Needs an even grid and an even number of M
// tiles, so the two CTAs' tile t and t + 1 always share an N tile.
// AT (fp4, bias-folded, 256 columns): the A ring lives in TMEM (tcgen05.st by
// the producers, `kind::mxf4` TS MMAs) and shared memory carries only B: per
// 128 x 256 tile the MMA's shared-memory reads drop from 432 to 288 KB and the
// producers' 144 KB of A stores leave shared memory — at the full MMA rate the
// SS form needed ~864 KB per 4,600-cycle tile against 128 B/clk
template <int BN, int AM, int EM, int NPW, int BKS, int NEPI, bool KS, bool F4, bool KB = false, bool MC = false,
          bool AT = false>
__global__ void __launch_bounds__(num_threads<NPW, NEPI>(), 1) k_tc_gemm(const __grid_constant__ CUtensorMap bmap,
                                                                  const __grid_constant__ CUtensorMap amap,
                                                                  const Args g) {
  constexpr bool ATMA = AM == A_BYTES_TMA;  // A by TMA into shared memory, no producer warps
  static_assert(!AT || (F4 && (KB || AM == A_ROWS) && BN == 256 && !KS && B2_KB_DRAIN2),
                "TMEM A ring: bias-folded conv or row 256-column fp4 kernels");
  constexpr bool ASMEM = (F4 && !AT) || ATMA;  // A ring in shared memory
  constexpr int WS = BKS / 32;        // K words per stage
  constexpr int HALVES = NPW >= 4 ? NPW / 4 : 1;  // producer warps per lane quarter
  constexpr int WPH = WS / HALVES;    // K words per producer thread per stage
  constexpr int A_STAGE_COLS = BKS / 4;
  constexpr int EPI0 = 4 + NPW;       // first epilogue warp
  static_assert(ATMA || WPH == 2 || WPH == 4 || WPH == 8, "producer word split");
  static_assert(!ATMA || (NPW == 0 && !F4 && !KS), "TMA-fed u8 rows: int8, no producers, no split-K");
  constexpr bool POOLED = (EM == E_POOLPACK);
  static_assert(!F4 || AM != A_BYTES, "u8 rows are not fp4 operands");
  constexpr int B_STAGE_BYTES = F4 ? BN * BKS / 2 : BN * BKS;
  constexpr int A_STAGE_BYTES = F4 ? BM * BKS / 2 : BM * BKS;  // A stage in shared memory (fp4 / TMA-fed u8)
  constexpr int KMMA = F4 ? 64 : 32;            // K per MMA instruction
  constexpr int VW = F4 ? 4 : 8;                // widened words per 32-bit input word
  // one ring: stage s = B tile in shared memory + A block in TMEM, one
  // full barrier (TMA bytes + producer warps) and one empty barrier (MMA
  // commit): the issuing thread's per-stage waits and commits are serial
  // time the tensor pipe cannot hide at N = 128 (tools/microbench/mma_loop.cu)
  constexpr int SA = AT     ? at_stages<BN, BKS>()
                     : F4     ? f4_stages<BN, BKS>()
                     : ATMA ? (192 * 1024) / (B_STAGE_BYTES + A_STAGE_BYTES)
                            : (a_stages<BN, AM, BKS>() < b_stages<BN, BKS>() ? a_stages<BN, AM, BKS>() : b_stages<BN, BKS>());
  constexpr int SB = SA;
  constexpr int ACC_COLS = BN;
  // TMA-fed u8: TMEM holds only accumulators (no scale factors for int8): double-buffered even at 256 columns
  constexpr int ACC_BUFS = F4 ? f4_acc_bufs<BN>() : ATMA ? (BN > 128 ? 2 : 3) : acc_bufs<BN, AM>();
  constexpr int A_COL0 = ACC_BUFS * ACC_COLS;  // i8: A ring; fp4: scale-factor columns
  constexpr int AR0 = A_COL0 + 2 * F4_SF_COLS;  // AT: the A ring after the scale and bias-scale columns
  constexpr int AR_STAGE = BKS / 8;             // AT: TMEM columns per stage (8 e2m1 per column)
  static_assert(!AT || AR0 + SA * AR_STAGE <= 512, "TMEM: accumulator, scales, A ring");
  static_assert(F4 ? (A_COL0 + F4_SF_COLS <= 512) : ATMA ? (A_COL0 <= 512) : (A_COL0 + SA * A_STAGE_COLS <= 512),
                "TMEM budget");
  constexpr uint32_t IDESC = F4 ? idesc_f4(BN) : idesc_i8(BN, AM == A_BYTES || ATMA);
  constexpr bool BIASK = KB;
  // H2 (TMEM-A-ring bias-folded 256-column kernels): the accumulator's two
  // 128-column halves get their own full / empty barriers, and each block of
  // H2_R K stages is issued half 0 first, then half 1 (N = 128 MMAs).  Half 0
  // completes H2_R stages before the tile does, so its drain overlaps the
  // last block's half-1 MMAs, and the next tile's first half-0 MMAs give the
  // epilogue that much time to drain half 1 (one 256-column accumulator:
  // the MMA thread had waited 17 % of conv4 for it)
  constexpr bool H2 = AT && KB && B2_H2 && BN == 256;
  constexpr int NTB = H2 ? 2 : ACC_BUFS;  // accumulator barrier pairs
  static_assert(!H2 || (NEPI == 8 && ACC_BUFS == 1 && !B2_EPI_ONE_POLLER), "H2: two epilogue warps per lane quarter");
  static_assert(!KB || (F4 && !KS && (EM == E_PACK || EM == E_POOLPACK)), "bias fold: packed fp4 output");
  static_assert(!MC || (F4 && !KS), "multicast weights: fp4, no split-K");
  static_assert(!BIASK || A_COL0 + 2 * F4_SF_COLS <= (ACC_BUFS == 1 ? 288 : 512), "TMEM: bias scale columns");
  constexpr int B_REGION = (ASMEM || AT) ? SB * B_STAGE_BYTES : b_stages<BN, BKS>() * B_STAGE_BYTES;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array (an
  // integer round trip would turn every table read into a generic load)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sb = smem;                                                      // SB x B_STAGE_BYTES
  // the B region is sized for b_stages() (a resident B tile may use all of it);
  // fp4: the A ring follows it
  uint8_t* sa = smem + B_REGION;
  int4* sthr = reinterpret_cast<int4*>(smem + B_REGION + (ASMEM ? SA * A_STAGE_BYTES : 0));  // THR_COLS/2 x (mul, add, ...)
  uint32_t* sgm = reinterpret_cast<uint32_t*>(sthr + THR_COLS / 2);        // THR_COLS/32 ge-direction masks
  uint64_t* full = reinterpret_cast<uint64_t*>(sgm + THR_COLS / 32);
  uint64_t* empty = full + SA;
  uint64_t* tfull = empty + SA;
  uint64_t* tempty = tfull + NTB;
  uint64_t* bres = tempty + NTB;  // resident-B load complete
  uint64_t* bbias = bres + 1;          // kbias: the bias block and the +1 block are written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bbias + 1);
  // kbias: the filters' bias blocks in the threshold table's place (no
  // swizzle, K-major: plane p = elements 32 p .. 32 p + 31 of every row, rows
  // 16 B apart, planes KB_COLS * 16 B apart) and a 128-row +1 block after the barriers
  uint8_t* sbias = reinterpret_cast<uint8_t*>(sthr);
  uint8_t* sones = reinterpret_cast<uint8_t*>(tmem_slot + 2);
  sones += (128u - (smem_u32(sones) & 127u)) & 127u;
  static_assert(KB_COLS * 32 <= THR_COLS * 8, "bias blocks fit the threshold table");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mtiles = (g.M + BM - 1) / BM;
  const int ntiles = (g.N + BN - 1) / BN;
  const int64_t tiles = mtiles * ntiles;  // tile t -> (m tile t % mtiles, n tile t / mtiles)
  // split-K (KS): the ksp K splits of a tile are the ranks of one cluster;
  // work item t -> tile t / ksp, split t % ksp; one item per CTA
  const int ksp = KS ? g.ksplit : 1;
  const int64_t items = tiles * ksp;
  const bool resb = !KS && g.resb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < SA; ++s) {
      // every A-producer warp (+ the TMA expect_tx arrival; TMA-fed A: that arrival only)
      mbar_init(&full[s], ATMA ? 1 : NPW + (resb ? 0 : 1));
      mbar_init(&empty[s], MC ? 2 : 1);  // MC: both CTAs' MMAs release the stage
    }
    mbar_init(bres, 1);
    mbar_init(bbias, 1);
    for (int a = 0; a < NTB; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], H2 ? NEPI / 2 : NEPI);  // H2: one barrier pair per 128-column half
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&bmap) : "memory");
    if constexpr (ATMA) asm volatile("prefetch.tensormap [%0];" ::"l"(&amap) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  if constexpr (MC)
    cluster_sync_all();  // the peer's barriers exist before any multicast or remote commit
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if constexpr (F4) {  // unit block scales (e8m0 0x7F = 2^0) for A and B, every lane
    if (warp < 4) {
      uint32_t ones[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) ones[i] = 0x7F7F7F7Fu;
      tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + A_COL0, ones);
      if constexpr (BIASK) {  // the bias blocks' B scales (every lane quarter holds all N rows)
#pragma unroll
        for (int i = 0; i < 16; ++i) ones[i] = PR_BIAS_SF;
        tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + A_COL0 + F4_SF_COLS, ones);
      }
      tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  // barriers, TMEM and the tensor map are set up while the previous kernel
  // drains; every global access (weights included: a widen may have just
  // written them) comes after the wait
  pdl_entry();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (B)
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      if constexpr ((AM == A_CONV || AM == A_ROWS) && !KS) {
        prefetch_tile_inputs<AM>(g, blockIdx.x, mtiles, tiles);
        prefetch_tile_inputs<AM>(g, blockIdx.x + gridDim.x, mtiles, tiles);
      }
      if (resb) {  // one N tile: load every K stage of B once, then only prefetch A inputs
        mbar_expect_tx(bres, (uint32_t)g.nkb * B_STAGE_BYTES);
        for (int kb = 0; kb < g.nkb; ++kb)
#pragma unroll
          for (int at = 0; at < (F4 ? BKS / 256 : BKS / BK); ++at)
            tma_load_2d(sb + kb * B_STAGE_BYTES + at * BN * BK, &bmap, bres, (F4 ? kb * BKS / 2 : kb * BKS) + at * BK, 0);
      }
      for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
        const int n0 = (int)(t / ksp / mtiles) * BN;
        if constexpr ((AM == A_CONV || AM == A_ROWS) && !KS)
          prefetch_tile_inputs<AM>(g, t + 2 * (int64_t)gridDim.x, mtiles, tiles);
        if (resb && !ATMA) continue;
        int kb0, kb1;
        item_krange(g, ksp, t, kb0, kb1);
        const int m0 = (int)((t % mtiles) * BM);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_nc(&empty[s], ph ^ 1);
          if constexpr (ATMA) {  // this stage's A boxes (u8 rows m0.., K bytes kb*BKS..), then B unless resident
            mbar_expect_tx(&full[s], A_STAGE_BYTES + (resb ? 0 : B_STAGE_BYTES));
#pragma unroll
            for (int at = 0; at < BKS / BK; ++at)
              tma_load_2d(sa + s * A_STAGE_BYTES + at * BM * BK, &amap, &full[s], kb * BKS + at * BK, m0);
            if (resb) {
              if (++s == SB) s = 0, ph ^= 1;
              continue;
            }
          } else {
            mbar_expect_tx(&full[s], B_STAGE_BYTES);
          }
          if constexpr (MC) {
            // this CTA's half of the rows, into both CTAs' stage s
            const uint32_t rk = cluster_rank_u();
#pragma unroll
            for (int at = 0; at < BKS / 256; ++at)
              tma_load_2d_mc(sb + s * B_STAGE_BYTES + at * BN * BK + rk * (BN / 2) * BK, &bmap, &full[s],
                             kb * BKS / 2 + at * BK, n0 + (int)rk * (BN / 2), (uint16_t)3);
          } else
#pragma unroll
          for (int at = 0; at < (F4 ? BKS / 256 : BKS / BK); ++at)  // one 128-byte-wide box per swizzle atom
            tma_load_2d(sb + s * B_STAGE_BYTES + at * BN * BK, &bmap, &full[s], (F4 ? kb * BKS / 2 : kb * BKS) + at * BK,
                        n0);
          if (++s == SB) s = 0, ph ^= 1;
        }
      }
    }
  } else if (BIASK && warp == 3) {
    // ------------------------------------------------ kbias: bias blocks + the +1 block, once
    {
      const int ncols = ((g.N + BN - 1) / BN) * BN;
      for (int n = lane; n < ncols; n += 32) {
        uint4 b0, b1;
        pr_bias_bytes(filter_bias(g.thresh, g.ge, n, g.N, g.kbias), b0, b1);
        *reinterpret_cast<uint4*>(sbias + n * 16) = b0;
        *reinterpret_cast<uint4*>(sbias + KB_COLS * 16 + n * 16) = b1;
      }
      for (int i = lane; i < 4096 / 16; i += 32)
        reinterpret_cast<uint4*>(sones)[i] = make_uint4(0x22222222u, 0x22222222u, 0x22222222u, 0x22222222u);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bbias);
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // (B2_TC_WARP_ISSUE: the whole warp runs the loop with uniform
    // descriptors, one elected lane issues — see tc_padrow.cuh)
    constexpr bool WI = B2_TC_WARP_ISSUE != 0 || AT || (F4 && B2_TC_WI_F4);  // AT: measured conv4 3.44 -> 3.30 ms with it
    if (WI || lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      if (resb) mbar_wait(bres, 0);
      bool bias_ready = false;
      const uint64_t ones_desc = BIASK ? noswz_desc_k(smem_u32(sones), 2048) : 0;
      const uint64_t bias_desc = BIASK ? noswz_desc_k(smem_u32(sbias), KB_COLS * 16) : 0;
      // warp-uniform TMEM base and B descriptor halves (the start-address
      // offsets of a stage only touch the descriptor's low word)
      const uint32_t tm = WI ? __shfl_sync(0xffffffffu, tmem, 0) : tmem;
      const uint64_t b0desc = sw128_desc(smem_u32(sb));
      const uint32_t b0_lo = (uint32_t)b0desc, b0_hi = (uint32_t)(b0desc >> 32);
#ifdef B2_TC_TIMING
      long long c_acc = 0, c_full = 0, c_t0 = clock64(), c_x;
#endif
      for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
        if constexpr (H2) {
          // half-ordered blocks of B2_H2_R stages (see H2 above)
          int kb0, kb1;
          item_krange(g, ksp, t, kb0, kb1);
          const int n0 = (int)((t / ksp) / mtiles) * BN;
          constexpr uint32_t IDESC128 = idesc_f4(128);
          for (int b = kb0; b < kb1; b += B2_H2_R) {
            const int nb = kb1 - b < B2_H2_R ? kb1 - b : B2_H2_R;
            int ss[B2_H2_R];
#pragma unroll
            for (int i = 0; i < B2_H2_R; ++i) {
              if (i < nb) {
                ss[i] = s;
#ifdef B2_TC_TIMING
                c_x = clock64();
#endif
                mbar_wait(&full[s], ph);
#ifdef B2_TC_TIMING
                c_full += clock64() - c_x;
#endif
                if (++s == SA) s = 0, ph ^= 1;
              }
            }
            tc_fence_after();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (b == kb0) {
#ifdef B2_TC_TIMING
                c_x = clock64();
#endif
                mbar_wait(&tempty[h], aph ^ 1);
#ifdef B2_TC_TIMING
                c_acc += clock64() - c_x;
#endif
                tc_fence_after();
              }
              if (pr_elect<WI>()) {
#pragma unroll
                for (int i = 0; i < B2_H2_R; ++i) {
                  if (i < nb) {
                    const int kmma = b + i + 1 == g.nkb ? g.klast : BKS / KMMA;
                    const uint32_t blo = b0_lo + (uint32_t)((ss[i] * B_STAGE_BYTES + h * 128 * BK) >> 4);
#pragma unroll
                    for (int k = 0; k < BKS / 64; ++k)
                      if (k < kmma)
                        tc_mma_f4_ts_g(tm + h * 128, tm + AR0 + ss[i] * AR_STAGE + k * 8,
                                       ((uint64_t)b0_hi << 32) |
                                           (blo + (uint32_t)(((k >> 2) * BN * BK + (k & 3) * 32) >> 4)),
                                       IDESC128, tm + A_COL0, tm + A_COL0 + 4, (b > kb0 || i || k) ? 1u : 0u);
                  }
                }
                if (b + nb == kb1) {  // the half's threshold block, then its accumulator is done
                  if (!bias_ready) mbar_wait(bbias, 0), bias_ready = true;
                  tc_mma_f4(tm + h * 128, ones_desc, bias_desc + (uint64_t)(((n0 + h * 128) * 16) >> 4), IDESC128,
                            tm + A_COL0, tm + A_COL0 + F4_SF_COLS, 1u);
                  tc_commit(&tfull[h]);
                }
              }
            }
            if (pr_elect<WI>()) {
#pragma unroll
              for (int i = 0; i < B2_H2_R; ++i)
                if (i < nb) {
                  if constexpr (MC)
                    tc_commit_mc(&empty[ss[i]], (uint16_t)3);
                  else
                    tc_commit(&empty[ss[i]]);
                }
            }
          }
          aph ^= 1;
          continue;
        }
#ifdef B2_TC_TIMING
        c_x = clock64();
#endif
        mbar_wait(&tempty[acc], aph ^ 1);
#ifdef B2_TC_TIMING
        c_acc += clock64() - c_x;
#endif
        tc_fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        int kb0, kb1;
        item_krange(g, ksp, t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
#ifdef B2_TC_TIMING
          c_x = clock64();
#endif
          mbar_wait(&full[s], ph);
#ifdef B2_TC_TIMING
          c_full += clock64() - c_x;
#endif
          tc_fence_after();
          const uint32_t bs = smem_u32(sb + (resb ? kb : s) * B_STAGE_BYTES);
          const int kmma = kb + 1 == g.nkb ? g.klast : BKS / KMMA;
          if constexpr (AT) {
            // A from the TMEM ring (8 columns per K=64), B in shared memory
            const uint32_t blo = b0_lo + (uint32_t)(((resb ? kb : s) * B_STAGE_BYTES) >> 4);
            const uint32_t dd = tm + acc * ACC_COLS;
            if (pr_elect<WI>()) {
#pragma unroll
              for (int k = 0; k < BKS / 64; ++k)
                if (k < kmma)
                  tc_mma_f4_ts_g(dd, tm + AR0 + s * AR_STAGE + k * 8,
                                 ((uint64_t)b0_hi << 32) | (blo + (uint32_t)(((k >> 2) * BN * BK + (k & 3) * 32) >> 4)),
                                 IDESC, tm + A_COL0, tm + A_COL0 + 4, (kb > kb0 || k) ? 1u : 0u);
            }
          } else if constexpr (F4) {
            // both operands in shared memory: 4 K=64 MMAs per 128-byte swizzle atom
            // (descriptors as uniform (lo + offset, hi), as the AT form)
            const uint64_t a0desc = sw128_desc(smem_u32(sa));
            const uint32_t alo = (uint32_t)a0desc + (uint32_t)((s * A_STAGE_BYTES) >> 4), a_hi = (uint32_t)(a0desc >> 32);
            const uint32_t blo = b0_lo + (uint32_t)(((resb ? kb : s) * B_STAGE_BYTES) >> 4);
            const uint32_t dd = tm + acc * ACC_COLS;
            if (pr_elect<WI>()) {
#pragma unroll
              for (int k = 0; k < BKS / 64; ++k)
                if (k < kmma)
                  tc_mma_f4(dd, ((uint64_t)a_hi << 32) | (alo + (uint32_t)(((k >> 2) * BM * BK + (k & 3) * 32) >> 4)),
                            ((uint64_t)b0_hi << 32) | (blo + (uint32_t)(((k >> 2) * BN * BK + (k & 3) * 32) >> 4)),
                            IDESC, tm + A_COL0, tm + A_COL0 + 4, (kb > kb0 || k) ? 1u : 0u);
            }
          } else if constexpr (ATMA) {
            // u8 A and s8 B both in shared memory (128-byte swizzle, K-major)
            const uint32_t as = smem_u32(sa + s * A_STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < BKS / 32; ++k)
              if (k < kmma && pr_elect<WI>())
                tc_mma_i8_ss(d, sw128_desc(as + (k >> 2) * BM * BK + (k & 3) * 32),
                             sw128_desc(bs + (k >> 2) * BN * BK + (k & 3) * 32), IDESC, (kb > kb0 || k) ? 1u : 0u);
          } else {
            const uint32_t a = tmem + A_COL0 + s * A_STAGE_COLS;
#pragma unroll
            for (int k = 0; k < BKS / 32; ++k)
              if (k < kmma && pr_elect<WI>())
                tc_mma_i8(d, a + k * 8, sw128_desc(bs + (k >> 2) * BN * BK + (k & 3) * 32), IDESC,
                          (kb > kb0 || k) ? 1u : 0u);
          }
          if (pr_elect<WI>()) {
            if constexpr (MC)
              tc_commit_mc(&empty[s], (uint16_t)3);
            else
              tc_commit(&empty[s]);
          }
          if (++s == SA) s = 0, ph ^= 1;
        }
        if constexpr (BIASK) {  // + the tile's columns' bias: A = +1 block, B = bias rows n0 ..
          if (!bias_ready) mbar_wait(bbias, 0), bias_ready = true;
          const int n0 = (int)((t / ksp) / mtiles) * BN;
          if (pr_elect<WI>())
            tc_mma_f4(d, ones_desc, bias_desc + (uint64_t)((n0 * 16) >> 4), IDESC, tmem + A_COL0,
                      tmem + A_COL0 + F4_SF_COLS, 1u);
        }
        if (pr_elect<WI>()) tc_commit(&tfull[acc]);
        if (++acc == ACC_BUFS) acc = 0, aph ^= 1;
      }
#ifdef B2_TC_TIMING
      if (blockIdx.x < 2 && lane == 0)
        printf("AM %d BN %d: total %lld  wait acc %lld  wait full %lld  items %lld\n", AM, BN, clock64() - c_t0, c_acc,
               c_full, (items - blockIdx.x + gridDim.x - 1) / gridDim.x);
#endif
    }
  } else if (warp >= 4 && warp < EPI0) {
    // ------------------------------------------------ A producers
    // Two warps per TMEM lane quarter, each producing half (64 elements) of
    // the row's 128-element K block.  The cursor runs PF K blocks ahead of
    // the stage being written (across tile boundaries), so the global
    // gathers overlap the widening and the TMEM stores; each stage is
    // published one iteration later, after its tcgen05.st has drained.
    const int q = warp & 3;
    const int half = HALVES == 1 ? 0 : (warp - 4) >> 2;
    const int r = q * 32 + lane;  // tile row = TMEM lane
    const uint32_t st_addr = tmem + ((uint32_t)(q * 32) << 16) + A_COL0 + half * (A_STAGE_COLS / HALVES);
    const uint32_t at_addr = tmem + ((uint32_t)(q * 32) << 16) + AR0 + half * (AR_STAGE / HALVES);  // AT
    constexpr bool CONV_FAST = AM == A_CONV && F4 && !KS && WPH == 4 && B2_CONV_FAST;
    ACursor<AM, POOLED, WS, WPH, F4 && AM == A_CONV> cur;
    cur.start(g, blockIdx.x, mtiles, tiles, r, half, ksp);
    int64_t jobs;
    if constexpr (KS) {
      jobs = 0;
      for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
        int kb0, kb1;
        item_krange(g, ksp, t, kb0, kb1);
        jobs += kb1 - kb0;
      }
    } else {
      const int64_t my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      jobs = my_tiles * g.nkb;
    }
    int s = 0, pending = -1;
    uint32_t ph = 0;
#ifdef B2_TC_TIMING
    long long p_wait = 0;
    const long long p_t0 = clock64();
#endif
    // every stage feeds exactly one K=32 MMA (K <= 32, one stage): the first
    // conv; only the first word of each producer's share is consumed
    const bool short_k = HALVES == 1 && g.nkb == 1 && g.klast == 1;
    auto publish = [&](int stage, uint32_t (&v)[VW * WPH]) {  // i8: WPH 2/4/8 -> 16/32/64 TMEM columns
      if constexpr (AT) {
        // fp4 A in TMEM: this thread's 4 words = 16 columns (column j = K
        // elements 8 j .. 8 j + 7) of its lane, published one stage later
        if (pending >= 0) {
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[pending]);
        }
#ifdef B2_TC_TIMING
        const long long pw0 = clock64();
#endif
        mbar_wait_nc(&empty[stage], ph ^ 1);
#ifdef B2_TC_TIMING
        p_wait += clock64() - pw0;
#endif
        tc_fence_after();
        static_assert(!AT || WPH == 4 || WPH == 2, "AT: 16 or 8 columns per producer thread");
        if constexpr (WPH == 4)
          tmem_st16(at_addr + stage * AR_STAGE, *reinterpret_cast<uint32_t(*)[16]>(v));
        else
          tmem_st8(at_addr + stage * AR_STAGE, v);
        if constexpr (B2_AT_EAGER) {  // publish now (the store's drain on this warp's critical path)
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[stage]);
          return;
        }
        pending = stage;
        return;
      } else if constexpr (F4) {
        // fp4: this thread's WPH words of the stage are WPH 16-byte chunks of
        // its row in the shared-memory A stage (128-byte swizzle, K-major)
        mbar_wait_nc(&empty[stage], ph ^ 1);
        uint8_t* row = sa + stage * A_STAGE_BYTES + r * 128;
        // one K stage per tile (the first conv): only the words its klast
        // K=64 MMAs read are stored
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
        if (lane == 0) mbar_arrive(&full[stage]);
        return;
      }
      if (pending >= 0) {
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[pending]);
      }
      mbar_wait_nc(&empty[stage], ph ^ 1);
      tc_fence_after();
#ifndef B2_PROBE_SKIP_A
      if constexpr (WPH == 8) {
        tmem_st32(st_addr + stage * A_STAGE_COLS, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_st32(st_addr + stage * A_STAGE_COLS + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      } else if constexpr (WPH == 4) {
        if (short_k)  // one K=32 MMA reads this stage: only its 8 columns matter
          tmem_st8(st_addr + stage * A_STAGE_COLS, v);
        else
          tmem_st32(st_addr + stage * A_STAGE_COLS, *reinterpret_cast<uint32_t(*)[32]>(v));
      } else {
        tmem_st16(st_addr + stage * A_STAGE_COLS, *reinterpret_cast<uint32_t(*)[16]>(v));
      }
#endif
      pending = stage;
    };
    if constexpr (AM == A_BYTES) {
      static_assert(NPW == 8 && WS == 4, "u8 rows: two producer warps per quarter, 128-element stages");
      uint4 qx[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        cur.fetch_bytes(g, half, qx[u]);
        cur.advance(g, gridDim.x, mtiles, tiles, r, half, ksp);
      }
      for (int64_t j0 = 0; j0 < jobs; j0 += 2) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (j0 + u < jobs) {
            uint32_t v[16];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              v[4 * i + 0] = qx[u][i].x;
              v[4 * i + 1] = qx[u][i].y;
              v[4 * i + 2] = qx[u][i].z;
              v[4 * i + 3] = qx[u][i].w;
            }
            cur.fetch_bytes(g, half, qx[u]);
            cur.advance(g, gridDim.x, mtiles, tiles, r, half, ksp);
            publish(s, v);
            if (++s == SA) s = 0, ph ^= 1;
          }
        }
      }
    } else if constexpr (WPH == 8) {
      // 512-element stages: two 4-word chunks per thread, widened and stored
      // as two 32-column TMEM writes
      constexpr int PF8 = 2;
      uint4 qx[PF8][2];
      bool qok[PF8][2];
#pragma unroll
      for (int u = 0; u < PF8; ++u) {
        cur.fetch_bits8(g, half, qx[u], qok[u]);
        cur.advance(g, gridDim.x, mtiles, tiles, r, half, ksp);
      }
      const int ijobs = (int)jobs;
      for (int j0 = 0; j0 < ijobs; j0 += PF8) {
#pragma unroll
        for (int u = 0; u < PF8; ++u) {
          if (j0 + u < ijobs) {
            uint32_t v[VW * 8];
#ifndef B2_PROBE_SKIP_A
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              if constexpr (F4) {
                widen_f4(qx[u][c].x, qok[u][c], v + 16 * c + 0);
                widen_f4(qx[u][c].y, qok[u][c], v + 16 * c + 4);
                widen_f4(qx[u][c].z, qok[u][c], v + 16 * c + 8);
                widen_f4(qx[u][c].w, qok[u][c], v + 16 * c + 12);
              } else {
                widen32(qx[u][c].x, qok[u][c], v + 32 * c + 0);
                widen32(qx[u][c].y, qok[u][c], v + 32 * c + 8);
                widen32(qx[u][c].z, qok[u][c], v + 32 * c + 16);
                widen32(qx[u][c].w, qok[u][c], v + 32 * c + 24);
              }
            }
#endif
            cur.fetch_bits8(g, half, qx[u], qok[u]);
            cur.advance(g, gridDim.x, mtiles, tiles, r, half, ksp);
            publish(s, v);
            if (++s == SA) s = 0, ph ^= 1;
          }
        }
      }
    } else if (CONV_FAST && g.kh * g.kw <= 32) {
      if constexpr (CONV_FAST) {
      // lean conv producer (ConvCursor): the same ring of PF prefetched
      // stages, flattened, with 32-bit shared addresses precomputed
      ConvCursor<POOLED, WS, WPH> cc;
      cc.start(g, blockIdx.x, mtiles, tiles, r, half);
      uint4 qx[PF];
      bool qok[PF];
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        cc.fetch(qx[u], qok[u]);
        cc.advance(g, gridDim.x, mtiles, tiles, r, half);
      }
      const uint32_t row0 = smem_u32(sa) + (uint32_t)r * 128u;
      const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
      uint32_t ck[4];  // this thread's four 16-byte chunks of its 128-byte row (swizzled)
#pragma unroll
      for (int i = 0; i < 4; ++i) ck[i] = (uint32_t)(((half * 4 + i) ^ (r & 7)) << 4);
      const int ijobs = (int)jobs;
      for (int j0 = 0; j0 < ijobs; j0 += PF) {
#pragma unroll
        for (int u = 0; u < PF; ++u) {
          if (j0 + u < ijobs) {
            uint32_t v[16];
            const uint32_t c2 = qok[u] ? 0xAAAAAAAAu : 0u;
            widen_f4x(qx[u].x, c2, v + 0);
            widen_f4x(qx[u].y, c2, v + 4);
            widen_f4x(qx[u].z, c2, v + 8);
            widen_f4x(qx[u].w, c2, v + 12);
            cc.fetch(qx[u], qok[u]);
            cc.advance(g, gridDim.x, mtiles, tiles, r, half);
            if constexpr (AT) {  // A ring in TMEM: the generic publish (tcgen05.st, published a stage later)
              publish(s, v);
              if (++s == SA) s = 0, ph ^= 1;
              continue;
            }
            mbar_wait_u(empty0 + 8u * (uint32_t)s, ph ^ 1);
            const uint32_t row = row0 + (uint32_t)s * (uint32_t)A_STAGE_BYTES;
#pragma unroll
            for (int i = 0; i < 4; ++i) sts128_u(row + ck[i], v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_u(full0 + 8u * (uint32_t)s);
            if (++s == SA) s = 0, ph ^= 1;
          }
        }
      }
      }
    } else {
      // BYTECONV keeps a per-bit validity word per slot; the row and conv
      // modes only a flag (valid rows widen to +/-1, invalid ones to 0)
      constexpr bool MASKED = AM == A_BYTECONV;
      uint4 qx[PF], qv[MASKED ? PF : 1];
      bool qok[PF];
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        uint4 vm;
        cur.template fetch_bits<WPH>(g, half, qx[u], vm);
        if constexpr (MASKED) qv[u] = vm;
        qok[u] = vm.x != 0 || vm.y != 0 || vm.z != 0 || vm.w != 0;
        cur.advance(g, gridDim.x, mtiles, tiles, r, half, ksp);
      }
      const int ijobs = (int)jobs;
      for (int j0 = 0; j0 < ijobs; j0 += PF) {
#pragma unroll
        for (int u = 0; u < PF; ++u) {
          if (j0 + u < ijobs) {
            uint32_t v[VW * WPH];
#ifndef B2_PROBE_SKIP_A
            if constexpr (F4) {
              if constexpr (MASKED) {
                widen_f4m(qx[u].x, qv[u].x, v + 0);
                widen_f4m(qx[u].y, qv[u].y, v + 4);
                if constexpr (WPH == 4) {
                  widen_f4m(qx[u].z, qv[u].z, v + 8);
                  widen_f4m(qx[u].w, qv[u].w, v + 12);
                }
              } else {
                widen_f4(qx[u].x, qok[u], v + 0);
                widen_f4(qx[u].y, qok[u], v + 4);
                if constexpr (WPH == 4) {
                  widen_f4(qx[u].z, qok[u], v + 8);
                  widen_f4(qx[u].w, qok[u], v + 12);
                }
              }
            } else if constexpr (MASKED) {
              widen32m(qx[u].x, qv[u].x, v + 0);
              if (!short_k) {
                widen32m(qx[u].y, qv[u].y, v + 8);
                if constexpr (WPH == 4) {
                  widen32m(qx[u].z, qv[u].z, v + 16);
                  widen32m(qx[u].w, qv[u].w, v + 24);
                }
              }
            } else {
              widen32(qx[u].x, qok[u], v + 0);
              widen32(qx[u].y, qok[u], v + 8);
              if constexpr (WPH == 4) {
                widen32(qx[u].z, qok[u], v + 16);
                widen32(qx[u].w, qok[u], v + 24);
              }
            }
#endif
            // refill the slot only after it was consumed: the load lands in
            // the same registers and nothing waits on it until PF stages later
            uint4 vm;
            cur.template fetch_bits<WPH>(g, half, qx[u], vm);
            if constexpr (MASKED) qv[u] = vm;
            qok[u] = vm.x != 0 || vm.y != 0 || vm.z != 0 || vm.w != 0;
            cur.advance(g, gridDim.x, mtiles, tiles, r, half, ksp);
            publish(s, v);
            if (++s == SA) s = 0, ph ^= 1;
          }
        }
      }
    }
    if (pending >= 0) {
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[pending]);
    }
#ifdef B2_TC_TIMING
    if (blockIdx.x < 1 && lane == 0 && (warp == 4 || warp == 8))
      printf("producer warp %d: total %lld  wait empty %lld\n", warp, clock64() - p_t0, p_wait);
#endif
  } else if (warp >= EPI0) {
    // ------------------------------------------------ epilogue
    constexpr int ECOLS = BN / (NEPI / 4);  // columns per epilogue warp
    constexpr int ECH = ECOLS / 32;         // 32-column chunks per epilogue warp
    // spare TMEM columns past the accumulators and scale factors (fp4, one
    // 256-column accumulator: columns 288..415 for the two warps of a lane
    // quarter) stage half of a warp's chunks during the drain
    constexpr int SPARE0 = 288;
    // (convolutions: measured 2-3 % faster, and the int32 GEMM; dense layers
    // with packed output were 7 % slower with it)
    constexpr bool STAGE_TMEM = F4 && (AM == A_CONV || EM == E_I32) && !KS && ECH == 4 && NEPI == 8 && ACC_BUFS == 1 &&
                                A_COL0 + F4_SF_COLS <= SPARE0 && SPARE0 + 2 * 64 <= 512 && B2_TMEM_STAGE;
    const int q = warp & 3;                 // EPI0 % 4 == 0: lane quarter
    const int r = q * 32 + lane;
    const int ec0 = ((warp - EPI0) >> 2) * ECOLS;  // first tile column of this warp
    const int et = (warp - EPI0) * 32 + lane;
    const uint32_t lane_addr = ((uint32_t)(q * 32) << 16) + ec0;
    int acc = 0;
    uint32_t aph = 0;
    // thresholds as bit = (acc * mul + add >= 0), resident for the launch
    // when all N columns fit the table, else staged per tile
    const int ncols = ntiles * BN;
    const bool static_thr = ncols <= THR_COLS;
    constexpr bool kb_on = BIASK;  // bias fold: sign bits, direction masks only
    if constexpr (EM == E_PACK || EM == E_POOLPACK) {
      if (static_thr) {
        stage_thresholds<F4>(g, 0, ncols, et, 32 * NEPI, lane, kb_on ? nullptr : sthr, sgm);
        epi_bar<NEPI>();
      }
    }
    if constexpr (KS) {
      // ---- split-K: reduce-scatter the ksp partial tiles over the cluster.
      // Rank `rank` owns tile rows [rank * rpo, +rpo); every rank writes its
      // partial of those rows into the owner's (now idle) B ring, slot
      // [source rank][row][RS], then each owner sums its rows and packs them.
      static_assert(EM == E_PACK || EM == E_POOLPACK, "split-K kernels pack their output");
      constexpr int RS = BN + 4;  // padded slot row (ints): conflict-free 16-byte reads across rows
      static_assert(BM * RS * 4 <= B_REGION, "reduction slots fit the B ring");
      const int64_t t = blockIdx.x;  // one item per CTA
      const int64_t tt = t / ksp;
      const int rank = (int)(t % ksp);
      const int rpo = BM / ksp;
      const int n0 = (int)(tt / mtiles) * BN;
      const int64_t mrow0 = (tt % mtiles) * BM + rank * rpo;  // first output row this rank owns
      int32_t* slots = reinterpret_cast<int32_t*>(sb);
      mbar_wait(&tfull[0], 0);
      tc_fence_after();
      cluster_sync_all();  // every rank's MMAs are done: all B rings are free
      {
        const int owner = r / rpo, lr = r % rpo;
        const uint32_t dst = cluster_map(smem_u32(slots + (rank * rpo + lr) * RS + ec0), (uint32_t)owner);
#pragma unroll
        for (int c = 0; c < ECH; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem + lane_addr + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            st_cluster_v4(dst + (c * 32 + 4 * i) * 4, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
      cluster_sync_all();  // all partials of my rows have landed
      const int units = rpo * (BN / 32);  // (row, 32-column chunk), rows fastest: a pool window = 4 lanes
      for (int u0 = 0; u0 < units; u0 += 32 * NEPI) {
        const int u = u0 + et;
        const bool act = u < units;
        const int row = act ? u % rpo : 0, chunk = act ? u / rpo : 0;
        uint32_t v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0;
        for (int src = 0; src < ksp; ++src) {
          const int4* p = reinterpret_cast<const int4*>(slots + (src * rpo + row) * RS + chunk * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int4 x = p[i];
            if constexpr (F4) {  // exact: integer-valued floats below 2^24
              v[4 * i] = __float_as_uint(__uint_as_float(v[4 * i]) + __int_as_float(x.x));
              v[4 * i + 1] = __float_as_uint(__uint_as_float(v[4 * i + 1]) + __int_as_float(x.y));
              v[4 * i + 2] = __float_as_uint(__uint_as_float(v[4 * i + 2]) + __int_as_float(x.z));
              v[4 * i + 3] = __float_as_uint(__uint_as_float(v[4 * i + 3]) + __int_as_float(x.w));
            } else {
              v[4 * i] += x.x, v[4 * i + 1] += x.y, v[4 * i + 2] += x.z, v[4 * i + 3] += x.w;
            }
          }
        }
        uint32_t w = thr_word<F4>(v, sthr + ((n0 + chunk * 32) >> 1));
        if constexpr (EM == E_POOLPACK) w = pool_word(w, sgm[(n0 >> 5) + chunk]);
        const int64_t m = mrow0 + row;
        const int wcol = n0 / 32 + chunk;
        if (act && m < g.M && (!POOLED || (row & 3) == 0) && wcol < g.ldo32)
          g.out_bits[(POOLED ? (m >> 2) : m) * g.ldo32 + wcol] = w;
      }
    } else
    for (int64_t t = blockIdx.x, mt = blockIdx.x % mtiles, nt = blockIdx.x / mtiles; t < tiles;
         t += gridDim.x, next_tile(mt, nt, gridDim.x, mtiles)) {
      const int64_t m = mt * BM + r;
      const int n0 = (int)nt * BN;
      const int tcol = static_thr ? n0 : 0;  // table column of this tile's first column
      const bool mok = m < g.M;
      if constexpr (EM == E_PACK || EM == E_POOLPACK) {
        if (!static_thr) {  // N too wide for the resident table: this tile's columns only
          epi_bar<NEPI>();
          stage_thresholds<F4>(g, n0, BN, et, 32 * NEPI, lane, sthr, sgm);
          epi_bar<NEPI>();
        }
      }
#ifdef B2_EPI_SLEEP
      mbar_wait_sleep(&tfull[acc], aph, B2_EPI_SLEEP);
#elif B2_EPI_ONE_POLLER
      // one warp polls the accumulator barrier, the others block on the
      // epilogue's named barrier (ncu: eight polling warps spent ~25 % of the
      // im2col kernel's issue slots spinning here)
      if (warp == EPI0) mbar_wait(&tfull[acc], aph);
      epi_bar<NEPI>();
#else
      mbar_wait_nc(&tfull[H2 ? ((warp - EPI0) >> 2) : acc], aph);
#endif
      tc_fence_after();
      uint32_t words[ECH];
      const int4* trow = sthr + ((tcol + ec0) >> 1);  // (mul, add) pairs of this warp's columns
      // TMEM -> registers.  Up to two chunks per warp: both loads in flight,
      // one wait, the accumulator goes back to the MMA before any math (the
      // single 256-column accumulator's drain is on the MMA's critical path);
      // more chunks: software-pipelined, chunk c + 1 in flight while chunk c
      // is processed (tcgen05.wait::ld waits for all prior loads)
      // per-chunk epilogue math on 32 accumulator columns held in v
      auto process = [&](const uint32_t (&v)[32], int c) {
        const int nb = n0 + ec0 + c * 32;
        if constexpr (EM == E_AFFINE) {
          // _kernels.py:285-295 bn_affine: three separately rounded IEEE
          // operations (no FMA contraction), bit-exact with numpy
          if (mok && nb < g.N) {
            double* o = g.out_f64 + m * g.ldo + nb;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = nb + j;
              if (n < g.N)
                o[j] = __dadd_rn(__dmul_rn(__dsub_rn((double)acc_int<F4>(v[j]), __ldg(g.mean + n)), __ldg(g.scale + n)),
                                 __ldg(g.beta + n));
            }
          }
        } else if constexpr (EM == E_I32) {
          if (mok && nb < g.N) {
            int32_t* o = g.out_i32 + m * g.ldo + nb;
            if (nb + 32 <= g.N && ((g.ldo & 3) == 0)) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<int4*>(o + j) = make_int4(acc_int<F4>(v[j]), acc_int<F4>(v[j + 1]),
                                                            acc_int<F4>(v[j + 2]), acc_int<F4>(v[j + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < g.N) o[j] = acc_int<F4>(v[j]);
            }
          }
        } else {
          uint32_t w;
          if constexpr (kb_on)
            w = sign_word(v) ^ sgm[((tcol + ec0) >> 5) + c];
          else
            w = thr_word<F4>(v, trow + c * 16);
          if constexpr (EM == E_POOLPACK) w = pool_word(w, sgm[((tcol + ec0) >> 5) + c]);
          words[c] = w;
        }
      };
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[H2 ? ((warp - EPI0) >> 2) : acc]);
      };
      const uint32_t abase = tmem + lane_addr + acc * ACC_COLS;
      uint32_t va[32], vb[32];
      if constexpr (STAGE_TMEM && (KB || AT) && B2_KB_DRAIN2) {
        // bias fold: a chunk collapses to its sign word at once (int32 output
        // with the A ring in TMEM: the spare columns are the ring), so the
        // drain is two TMEM round trips with the first pair processed in between
        tmem_ld32(abase, va);
        tmem_ld32(abase + 32, vb);
        tmem_wait_ld();
        process(va, 0);
        process(vb, 1);
        tmem_ld32(abase + 64, va);
        tmem_ld32(abase + 96, vb);
        tmem_wait_ld();
        release();
        process(va, 2);
        process(vb, 3);
      } else if constexpr (STAGE_TMEM) {
        // single 256-column accumulator (its drain stalls the MMA): copy the
        // first two chunks into this warp's spare TMEM columns, load the last
        // two, release — three TMEM round trips instead of four loads
        // separated by the threshold math — then work from registers / spare
        const uint32_t spare = tmem + ((uint32_t)(q * 32) << 16) + SPARE0 + ((warp - EPI0) >> 2) * 64;
        tmem_ld32(abase, va);
        tmem_ld32(abase + 32, vb);
        tmem_wait_ld();
        tmem_st32(spare, va);
        tmem_st32(spare + 32, vb);
        tmem_wait_st();
        tmem_ld32(abase + 64, va);
        tmem_ld32(abase + 96, vb);
        tmem_wait_ld();
        release();
        process(va, 2);
        process(vb, 3);
        tmem_ld32(spare, va);
        tmem_ld32(spare + 32, vb);
        tmem_wait_ld();
        process(va, 0);
        process(vb, 1);
      } else if constexpr (ECH <= 2) {
        // both chunks in flight, one wait, the accumulator goes back before any math
        tmem_ld32(abase, va);
        if (ECH == 2) tmem_ld32(abase + 32, vb);
        tmem_wait_ld();
        release();
        process(va, 0);
        if (ECH == 2) process(vb, 1);
      } else {
        // software-pipelined: chunk c + 1 in flight while chunk c is processed
        tmem_ld32(abase, va);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < ECH; ++c) {
          uint32_t(&v)[32] = (c & 1) ? vb : va;
          uint32_t(&vn)[32] = (c & 1) ? va : vb;
          if (c + 1 < ECH) tmem_ld32(abase + (c + 1) * 32, vn);
          process(v, c);
          if (c + 1 < ECH) tmem_wait_ld();
          if (c + 2 == ECH) release();  // every chunk is in registers: hand the accumulator back
        }
      }
      if constexpr (EM == E_PACK || EM == E_POOLPACK) {
        const int64_t site = POOLED ? (m >> 2) : m;
        const bool writer = mok && (!POOLED || (lane & 3) == 0);
        if (writer) {
          const int w0 = (n0 + ec0) / 32;
          uint32_t* o = g.out_bits + site * g.ldo32 + w0;
          // vector stores sized to this warp's words (w0 is a multiple of ECH;
          // ldo32 is always even: lines are whole uint64 words)
          if constexpr (ECH % 4 == 0) {
            if (w0 + ECH <= g.ldo32 && (g.ldo32 & 3) == 0) {
#pragma unroll
              for (int c = 0; c < ECH; c += 4)
                *reinterpret_cast<uint4*>(o + c) = make_uint4(words[c], words[c + 1], words[c + 2], words[c + 3]);
              goto stored;
            }
          } else if constexpr (ECH % 2 == 0) {
            if (w0 + ECH <= g.ldo32) {
#pragma unroll
              for (int c = 0; c < ECH; c += 2) *reinterpret_cast<uint2*>(o + c) = make_uint2(words[c], words[c + 1]);
              goto stored;
            }
          }
          {
#pragma unroll
            for (int c = 0; c < ECH; ++c)
              if (w0 + c < g.ldo32) o[c] = words[c];
          }
        stored:;
        }
      }
      if (++acc == ACC_BUFS) acc = 0, aph ^= 1;
    }
  }

  if constexpr (KS) {
    if (warp < EPI0) {  // the epilogue's two cluster barriers count every thread of every rank
      cluster_sync_all();
      cluster_sync_all();
    }
  }
  tc_fence_before();
  if constexpr (MC)
    cluster_sync_all();  // no CTA leaves while its peer can still multicast into it or commit to its barriers
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int BN, int BKS>
constexpr int smem_bytes_at() {  // fp4, A ring in TMEM: B stages only (+ table, barriers, bias extras)
  return at_stages<BN, BKS>() * BN * BKS / 2 + THR_COLS * 8 + THR_COLS / 8 + 8 * (2 * at_stages<BN, BKS>() + 8) + 16 +
         128 + 4096 + 1024;
}
template <int BN, int AM, int BKS, bool F4 = false>
constexpr int smem_bytes() {
  if constexpr (AM == A_BYTES_TMA)
    return (192 * 1024) / ((BN + BM) * BKS) * (BN + BM) * BKS + THR_COLS * 8 + THR_COLS / 8 + 8 * (2 * 8 + 11) + 16 +
           1024;
  else if constexpr (F4)
    return f4_stages<BN, BKS>() * (BN + BM) * BKS / 2 + THR_COLS * 8 + THR_COLS / 8 +
           8 * (2 * f4_stages<BN, BKS>() + 8) + 16 + 128 + 4096 + 1024;  // (+ bbias, the kbias +1 block)
  else
    return b_stages<BN, BKS>() * BN * BKS + THR_COLS * 8 + THR_COLS / 8 + 8 * (2 * a_stages<BN, AM, BKS>() + 7) +
           16 + 1024;
}

}  // namespace tc
}  // namespace b2
