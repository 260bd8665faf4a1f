// Host side of the tcgen05 binary GEMM (tc_i8.cuh): weight widening, TMA
// descriptors, persistent launches, and the C-ABI entry points of the
// tensor-core path (include/bitnn_b200.h, "tensor-core path").
#include <cudaTypedefs.h>

#include <mutex>

#include <stdlib.h>

#include "tc_i8.cuh"
#include "tc_padrow.cuh"
#include "tc_byteconv.cuh"
#include "tc_pair.cuh"

#ifndef B2_RESIDENT_B
#define B2_RESIDENT_B 1
#endif
#ifndef B2_NPW128  // producer warps of 128-column tiles
#define B2_NPW128 8
#endif
#ifndef B2_BKS128  // K elements per stage of 128-column tiles
#define B2_BKS128 512
#endif
#ifndef B2_SPLITK  // cluster split-K for few-tile launches (0: off)
#define B2_SPLITK 1
#endif
#ifndef B2_SMALLM_TILES  // below this many 256-column tiles use 128-column ones (0: never)
#define B2_SMALLM_TILES 74
#endif
#ifndef B2_BYTES_BN128  // Input8 (u8 rows) on 128-column tiles
#define B2_BYTES_BN128 0
#endif
#ifndef B2_NEPI_F4_256  // epilogue warps of fp4 256-column tiles (one accumulator: the drain stalls the MMA)
#define B2_NEPI_F4_256 8
#endif
#ifndef B2_NPW_F4_256  // producer warps of the 256-column fp4 kernels
#define B2_NPW_F4_256 8
#endif
#ifndef B2_NEPI_F4_128  // epilogue warps of fp4 128-column dense tiles (MMAs twice as fast: drain faster)
#define B2_NEPI_F4_128 8
#endif
#ifndef B2_NEPI_BYTECONV  // epilogue warps of the first conv (one K block per tile)
#define B2_NEPI_BYTECONV 8
#endif

namespace b2 {
namespace tc {

// _kernels.py:57-64 unpack_lines, widened to int8 for the tensor pipe:
// out[r, k] = bit ? +1 : -1 for k < K, 0 for K <= k < kpad.  With `permute`
// K is permuted inside each 32-element group exactly like the A-side
// widen32 (perm_pos); without it (u8 A operand) K stays in order.
__global__ void k_expand_i8(const uint64_t* __restrict__ w, int64_t rows, int64_t wpl, int64_t k, int64_t kpad,
                            int permute, int8_t* __restrict__ out) {
  pdl_entry();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one thread per 4 output bytes
  int64_t per_row = kpad / 4;
  if (t >= rows * per_row) return;
  int64_t r = t / per_row, k0 = (t - r * per_row) * 4;
  uint32_t word = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int64_t kk = k0 + j;
    if (permute) {
      const int pos = (int)(kk & 31);
      kk = (kk & ~int64_t(31)) + 8 * (pos & 3) + (pos >> 2);  // inverse of perm_pos
    }
    uint32_t b = 0;
    if (kk < k) b = ((w[r * wpl + (kk >> 6)] >> (kk & 63)) & 1ull) ? 0x01u : 0xFFu;
    word |= b << (8 * j);
  }
  reinterpret_cast<uint32_t*>(out)[t] = word;
}

// Weights for the fp4 path (kind::mxf4): out[r] = kpad/2 bytes of e2m1
// nibbles, +1.0 (0x2) / -1.0 (0xA) for the bits of K, 0 beyond; 16 bytes
// per 32-element group in the A side's permuted order (widen_f4m).  One
// thread per output word.
__global__ void k_expand_f4(const uint64_t* __restrict__ w, int64_t rows, int64_t wpl, int64_t k, int64_t kpad,
                            uint32_t* __restrict__ out) {
  pdl_entry();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_row = kpad / 8;  // output words
  if (t >= rows * per_row) return;
  const int64_t r = t / per_row, o = t - r * per_row;
  const int64_t j = o >> 2;  // 32-element group
  const int q = (int)(o & 3);
  uint32_t x = 0, valid = 0;
  const int64_t rem = k - 32 * j;
  if (rem > 0) {
    x = (uint32_t)(w[r * wpl + (j >> 1)] >> (32 * (j & 1)));
    valid = rem >= 32 ? ~0u : ((1u << rem) - 1u);
  }
  out[t] = (0xAAAAAAAAu ^ ((x << (3 - q)) & 0x88888888u)) & (((valid >> q) & 0x11111111u) * 0xFu);
}

// network.py:128-138 _PackedByteBN on the raw image followed by the bit
// im2col of _kernels.py:170-199 (unroll_packed): row = kw32 words of window
// bits (K order (dy, dx, c), c fastest) then kw32 words of validity (0 for
// window cells in the padding ring, so the tensor cores see zero padding
// and no correction map is needed).  Rows are ordered like the conv output
// (pool-window-major when `pooled`).
//
// One CTA per (image, band of BAND output rows): the byte batchnorm code of
// every input site the band touches (c <= 8 bits) is computed once into
// shared memory, then each thread assembles its pixels' windows from there.
// output rows per CTA of the first-conv unroll: 32 when the batch fills the
// GPU (fewer, fuller CTAs: 6 % faster at batch 8192), 8 for small batches
// (batch 1: four CTAs per image instead of one)
constexpr int BAND = 32, BAND_SMALL = 8;

__device__ __forceinline__ int64_t unroll_row(int64_t img, int oy, int ox, int ho, int wo, int pooled) {
  if (!pooled) return (img * ho + oy) * (int64_t)wo + ox;
  const int wp = wo >> 1;
  const int q = (oy >> 1) * wp + (ox >> 1);
  return img * (int64_t)ho * wo + 4 * q + 2 * (oy & 1) + (ox & 1);
}

// KH/KW/C > 0: compile-time window (fully unrolled, one 32-bit word when
// KH*KW*C <= 32); 0: runtime shape.
template <int KH, int KW, int C>
__global__ void __launch_bounds__(256) k_byte_unroll(const uint8_t* __restrict__ x, int h, int w, int c_, int kh_,
                                                     int kw_, int stride, int pad, int ho, int wo, int kw32,
                                                     int pooled, int band, const int32_t* __restrict__ t,
                                                     const uint8_t* __restrict__ ge, uint32_t* __restrict__ out) {
  pdl_entry();
  const int c = C ? C : c_, kh = KH ? KH : kh_, kw = KW ? KW : kw_;
  extern __shared__ uint8_t codes[];  // [in_rows][w]
  const int bands = (ho + band - 1) / band;  // grid = images x bands, flattened (no 65535 cap)
  const int64_t img = blockIdx.x / bands;
  const int oy0 = (int)(blockIdx.x % bands) * band;
  const int oy1 = min(oy0 + band, ho);
  const int iy0 = oy0 * stride - pad;
  const int in_rows = (oy1 - 1 - oy0) * stride + kh;
  const uint8_t* xi = x + img * (int64_t)h * w * c;
  int32_t tc[8];
  bool gc[8];
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    tc[ch] = ch < c ? __ldg(t + ch) : 0;
    gc[ch] = ch < c ? __ldg(ge + ch) != 0 : true;
  }
  for (int i = threadIdx.x; i < in_rows * w; i += blockDim.x) {
    const int iy = iy0 + i / w, ix = i % w;
    uint32_t code = 0;
    if (iy >= 0 && iy < h) {
      const uint8_t* px = xi + ((int64_t)iy * w + ix) * c;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        if (ch < c) code |= (uint32_t)thr_bit((int32_t)px[ch], tc[ch], gc[ch]) << ch;
    }
    codes[i] = (uint8_t)code;
  }
  __syncthreads();
  const uint32_t cmask = (1u << c) - 1u;
  if constexpr (KH > 0 && KW > 0 && C > 0 && KH * KW * C <= 32) {
    for (int p = threadIdx.x; p < (oy1 - oy0) * wo; p += blockDim.x) {
      const int oy = oy0 + p / wo, ox = p - (p / wo) * wo;
      uint32_t bits = 0, valid = 0;
#pragma unroll
      for (int dy = 0; dy < KH; ++dy) {
        const int iy = oy * stride + dy - pad;
        if (iy < 0 || iy >= h) continue;
        const uint8_t* srow = codes + (iy - iy0) * w;
#pragma unroll
        for (int dx = 0; dx < KW; ++dx) {
          const int ix = ox * stride + dx - pad;
          if (ix < 0 || ix >= w) continue;
          bits |= (uint32_t)srow[ix] << ((dy * KW + dx) * C);
          valid |= cmask << ((dy * KW + dx) * C);
        }
      }
      reinterpret_cast<uint2*>(out)[unroll_row(img, oy, ox, ho, wo, pooled)] = make_uint2(bits, valid);
    }
    return;
  }
  for (int p = threadIdx.x; p < (oy1 - oy0) * wo; p += blockDim.x) {
    const int oy = oy0 + p / wo, ox = p % wo;
    uint32_t bits[4] = {0, 0, 0, 0}, valid[4] = {0, 0, 0, 0};
    int pos = 0;
    for (int dy = 0; dy < kh; ++dy) {
      const int iy = oy * stride + dy - pad;
      const int srow = (iy - iy0) * w;
      for (int dx = 0; dx < kw; ++dx, pos += c) {
        const int ix = ox * stride + dx - pad;
        if (iy < 0 || iy >= h || ix < 0 || ix >= w) continue;
        const uint32_t code = codes[srow + ix];
        const int wd = pos >> 5, sh = pos & 31;
        bits[wd] |= code << sh;
        valid[wd] |= cmask << sh;
        if (sh + c > 32) {  // a site straddling two words
          bits[wd + 1] |= code >> (32 - sh);
          valid[wd + 1] |= cmask >> (32 - sh);
        }
      }
    }
    uint32_t* o = out + unroll_row(img, oy, ox, ho, wo, pooled) * 2 * kw32;
    for (int i = 0; i < kw32; ++i) {
      o[i] = bits[i];
      o[kw32 + i] = valid[i];
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// int8 (rows, kpad) K-major weights -> TMA map with (128 B x BN rows) boxes,
// 128-byte swizzle (the UMMA K-major SW128 canonical layout).
static int make_bmap(CUtensorMap* map, const int8_t* b, int64_t rows, int64_t kpad, int bn) {
  auto fn = encode_fn();
  if (!fn) return B2_EINVAL;
  cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kpad};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)bn};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(b), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : B2_EINVAL;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

#ifndef B2_MC_ROWS  // the int32 row GEMM (bgemm) shares weight stages between CTA pairs too
#define B2_MC_ROWS 0  // measured no faster (bgemm 8192: 3.79 vs 3.83 P ops/s)
#endif
// the multicast-weights instantiation exists for the bias-folded fp4 conv kernels
template <bool F4, bool KS, int EM, int AM>
constexpr bool KBP_MC() {
  return F4 && !KS && (EM == E_PACK || EM == E_POOLPACK) && AM == A_CONV;
}

// KS: split-K over thread-block clusters of g.ksplit CTAs (one tile's K
// splits), one work item per CTA.
template <int BN, int AM, int EM, int NPW, int BKS, int NEPI = (BN > 128 ? 8 : 4), bool KS = false, bool F4 = false>
int launch_bn(Args g, const int8_t* b_i8, int64_t kpad, int64_t k, cudaStream_t st, const CUtensorMap* amap = nullptr) {
  // fp32 accumulators: exact integers below 2^24; the epilogue's float -> int
  // conversion (acc_int) needs |dot| < 2^22
  if (F4 && k > (int64_t(1) << 22)) return B2_EINVAL;
  g.nkb = (int)((k + BKS - 1) / BKS);
  g.klast = (int)(((k - 1) % BKS) / (F4 ? 64 : 32) + 1);
  // one N tile whose every K stage fits the B ring space: keep it resident
  const int b_room = F4                    ? f4_stages<BN, BKS>()
                     : AM == A_BYTES_TMA ? (192 * 1024) / ((BN + BM) * BKS)
                                         : b_stages<BN, BKS>();
  g.resb = (!KS && g.N <= BN && g.nkb <= b_room && B2_RESIDENT_B) ? 1 : 0;
  // fp4 packed output: fold the thresholds into one more MMA per tile (the
  // bias magnitude |T| + 1 <= K + 1 must fit the two-block encoding)
  static const int kb_env = [] {
    const char* e = getenv("B2_KBIAS");
    return e ? atoi(e) : 1;
  }();
  g.kbias = (F4 && !KS && (EM == E_PACK || EM == E_POOLPACK) && kb_env &&
             (int64_t)((g.N + BN - 1) / BN) * BN <= KB_COLS && k <= 5760)
                ? (int)k
                : 0;
  // weight stages shared by CTA pairs (TMA multicast): streamed B (not
  // resident), bias-folded conv kernels, enough tiles for every SM, an even
  // number of M tiles (a pair's tiles t, t + 1 share their N tile)
  // (off by default: with the TMEM A ring and the warp-wide issue it measured
  // 3-4 % slower on conv4 and equal on conv5/conv6; B2_MCAST=1 opts in)
  static const int mc_env = [] {
    const char* e = getenv("B2_MCAST");
    return e ? atoi(e) : 0;
  }();
  const int64_t mt_count = (g.M + BM - 1) / BM;
  const bool mc_geom = !g.resb && mc_env && mt_count % 2 == 0 && mt_count * ((g.N + BN - 1) / BN) >= num_sms() &&
                       num_sms() % 2 == 0;
  // the int32 row GEMM (bgemm) shares weight stages only with the TMEM A ring below
  const bool mc = mc_geom && ((KBP_MC<F4, KS, EM, AM>() && g.kbias) ||
                              (F4 && !KS && BN == 256 && AM == A_ROWS && EM == E_I32 && B2_MC_ROWS));
  CUtensorMap map;
  if (int rc = make_bmap(&map, b_i8, g.N, F4 ? kpad / 2 : kpad, mc ? BN / 2 : BN)) return rc;
  constexpr bool KBP = F4 && !KS && (EM == E_PACK || EM == E_POOLPACK);
  // fp4 A ring in TMEM (k_tc_gemm AT): the 256-column bias-folded conv kernels
  constexpr bool ATP = F4 && !KS && BN == 256 &&
                      ((AM == A_CONV && (EM == E_PACK || EM == E_POOLPACK)) ||
                       (AM == A_ROWS && (EM == E_I32 || EM == E_PACK)));
  static const int at_env = [] {
    const char* e = getenv("B2_F4_ATMEM");
    return e ? atoi(e) : 1;
  }();
  const bool at = ATP && (g.kbias || AM == A_ROWS) && !g.resb && at_env;
  constexpr bool MCP = (KBP_MC<F4, KS, EM, AM>() || (AM == A_ROWS && EM == E_I32)) && ATP;
  if (mc && !at && AM == A_ROWS) return B2_EINVAL;  // (no shared-memory multicast row GEMM instantiated)
  // (the KB instantiation only with the bias block actually folded: its
  // writer fills KB_COLS columns, a wider N would overrun the block)
  auto kern = at && mc      ? k_tc_gemm<BN, AM, EM, NPW, BKS, NEPI, KS, F4, KBP, MCP, ATP>
              : at && g.kbias ? k_tc_gemm<BN, AM, EM, NPW, BKS, NEPI, KS, F4, KBP, false, ATP>
              : at          ? k_tc_gemm<BN, AM, EM, NPW, BKS, NEPI, KS, F4, false, false, (ATP && AM == A_ROWS)>
              : mc          ? k_tc_gemm<BN, AM, EM, NPW, BKS, NEPI, KS, F4, KBP, KBP_MC<F4, KS, EM, AM>()>
              : KBP && g.kbias ? k_tc_gemm<BN, AM, EM, NPW, BKS, NEPI, KS, F4, KBP>
                             : k_tc_gemm<BN, AM, EM, NPW, BKS, NEPI, KS, F4, false>;
  const int smem = at ? smem_bytes_at<BN, BKS>() : smem_bytes<BN, AM, BKS, F4>();
  static std::atomic<uint64_t> attr[6];  // one opt-in record per kernel instantiation chosen above
  smem_optin(kern, smem, attr[at ? (mc ? 4 : g.kbias ? 3 : 5) : mc ? 2 : g.kbias ? 1 : 0]);
  int64_t tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  CUtensorMap amap_v;  // A_BYTES_TMA: the u8 rows; unused otherwise
  if (amap)
    amap_v = *amap;
  else
    memset(&amap_v, 0, sizeof(amap_v));
  if constexpr (KS) {
    launch_kc(g.ksplit, kern, (unsigned)(tiles * g.ksplit), num_threads<NPW, NEPI>(), smem, st, map, amap_v, g);
  } else {
    g.ksplit = 1;
    int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    if (mc)
      launch_kc(2, kern, (unsigned)grid, num_threads<NPW, NEPI>(), smem, st, map, amap_v, g);
    else
      launch_k(kern, grid, num_threads<NPW, NEPI>(), smem, st, map, amap_v, g);
  }
  return launched();
}

// CTA-pair kernel (tc_pair.cuh): 256 x 256 tiles over two SMs, a third less
// shared-memory traffic per MAC than the single-CTA 128 x 256 tile.
#ifndef B2_PAIR
#define B2_PAIR 0  // measured slower than the single-CTA kernel; B2_PAIR=1 opts in
#endif
inline bool pair_on() {
  static const int on = [] {
    const char* e = getenv("B2_PAIR");
    return e ? atoi(e) : B2_PAIR;
  }();
  return on != 0;
}
template <int AM, int EM>
int launch_pair(Args g, const int8_t* b, int64_t kpad, int64_t k, cudaStream_t st) {
  if (k > (int64_t(1) << 22)) return B2_EINVAL;  // see launch_bn
  g.nkb = (int)((k + PAIR_BKS - 1) / PAIR_BKS);
  g.klast = (int)(((k - 1) % PAIR_BKS) / 64 + 1);
  g.resb = 0;
  g.ksplit = 1;
  CUtensorMap map;
  if (int rc = make_bmap(&map, b, g.N, kpad / 2, PAIR_BN / 2)) return rc;
  auto kern = k_pair_gemm<AM, EM>;
  constexpr int smem = pair_smem_bytes();
  static std::atomic<uint64_t> attr{0};
  smem_optin(kern, smem, attr);
  const int64_t tiles = ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + PAIR_BN - 1) / PAIR_BN);
  const int64_t pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
  launch_kc(2, kern, (unsigned)(2 * pairs), 32 * (4 + PAIR_NPW + PAIR_NEPI), smem, st, map, g);
  return launched();
}

// Split-K for launches with few tiles (small batches) and deep K: the ks K
// splits of each 128x128 tile run as one cluster and reduce over distributed
// shared memory, so the serial K walk of a deep layer spreads over ks SMs.
// Returns the split count (0: not applicable).
template <int AM, int EM>
int splitk_count(const Args& g, int64_t k) {
  if constexpr ((EM == E_PACK || EM == E_POOLPACK) && (AM == A_ROWS || AM == A_CONV)) {
    static const int on = [] {
      const char* e = getenv("B2_SPLITK");
      return e ? atoi(e) : B2_SPLITK;
    }();
    if (!on) return 0;
    if (AM == A_CONV && g.spw % 4 != 0) return 0;
    const int64_t ntiles = (g.N + 127) / 128;
    const int64_t tiles = ((g.M + BM - 1) / BM) * ntiles;
    const int64_t nkb = (k + 511) / 512;
    // the cluster launch, its two barriers and the exchange cost ~3 us
    // (measured, graph-replayed): worth it only for long K walks
    if (nkb < 8 || ntiles * 128 > THR_COLS || 2 * tiles > num_sms()) return 0;
    for (int ks = 8; ks >= 2; ks /= 2)
      if (ks <= nkb && tiles * ks <= num_sms()) return ks;
  }
  return 0;
}

// N <= 128: 128-column tiles, double-buffered accumulator, 512-element K
// stages (16 MMAs of 64 cycles per stage hide the issuing thread's per-stage
// wait + commit, tools/microbench/mma_loop.cu) (128-element when a producer's 4 words would straddle two conv
// sites, for u8 rows, and for the one-block first conv); otherwise 256-column
// tiles (one M=128 x N=256 MMA per 32 K: half the A widening per MAC) with
// 128-element stages.  Two producer warps per TMEM lane quarter, one for the
// first conv.
// fp4 operands (kind::mxf4, both from shared memory): 256-column tiles with
// 256-element stages (4 K=64 MMAs of 128 cycles), 128-column tiles with
// 512-element stages (8 of 64 cycles), three accumulator buffers; C = 64
// convolutions take 16 producer warps (two words per thread: a site is two
// words).
template <int AM, int EM>
int launch_f4(Args g, const int8_t* b, int64_t kpad, cudaStream_t st, int64_t k) {
  if constexpr (AM == A_BYTES) {
    return B2_EINVAL;
  } else {
    const bool two_words = AM == A_CONV && g.spw % 4 != 0;
    if (!two_words) {
      if (int ks = splitk_count<AM, EM>(g, k)) {
        if constexpr ((EM == E_PACK || EM == E_POOLPACK) && (AM == A_ROWS || AM == A_CONV)) {
          g.ksplit = ks;
          return launch_bn<128, AM, EM, 8, 512, 4, true, true>(g, b, kpad, k, st);
        }
      }
    }
    if constexpr (AM == A_BYTECONV) {
      return launch_bn<128, AM, EM, 8, 256, B2_NEPI_BYTECONV, false, true>(g, b, kpad, k, st);
    } else {
      if constexpr (AM == A_CONV) {
        if (two_words) {
          if (g.N > 128) return launch_bn<256, AM, EM, 16, 256, 8, false, true>(g, b, kpad, k, st);
          return launch_bn<128, AM, EM, 16, 256, 4, false, true>(g, b, kpad, k, st);
        }
      }
      if (g.N > 128) {
        const int64_t tiles256 = ((g.M + BM - 1) / BM) * ((g.N + 255) / 256);
        if (B2_SMALLM_TILES && tiles256 < B2_SMALLM_TILES)
          return launch_bn<128, AM, EM, 8, 512, 4, false, true>(g, b, kpad, k, st);
        // enough 256 x 256 tiles for every SM pair: the CTA-pair kernel
        if constexpr (AM == A_ROWS || AM == A_CONV) {
          if (pair_on() && ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + 255) / 256) >= num_sms() / 2)
            return launch_pair<AM, EM>(g, b, kpad, k, st);
        }
        return launch_bn<256, AM, EM, B2_NPW_F4_256, 256, B2_NEPI_F4_256, false, true>(g, b, kpad, k, st);
      }
      if constexpr (AM == A_ROWS) return launch_bn<128, AM, EM, 8, 512, B2_NEPI_F4_128, false, true>(g, b, kpad, k, st);
      return launch_bn<128, AM, EM, 8, 512, 4, false, true>(g, b, kpad, k, st);
    }
  }
}

template <int AM, int EM, bool F4 = false>
int launch(Args g, const int8_t* b_i8, int64_t kpad, cudaStream_t st, int64_t k, const CUtensorMap* amap = nullptr) {
  if (g.M == 0 || g.N == 0) return 0;
  if constexpr (F4) return launch_f4<AM, EM>(g, b_i8, kpad, st, k);
  if constexpr (AM == A_BYTES_TMA) {
    if (g.N > 128) return launch_bn<256, AM, EM, 0, 128, 8>(g, b_i8, kpad, k, st, amap);
    return launch_bn<128, AM, EM, 0, 128, 4>(g, b_i8, kpad, k, st, amap);
  } else {
  if (int ks = splitk_count<AM, EM>(g, k)) {
    if constexpr ((EM == E_PACK || EM == E_POOLPACK) && (AM == A_ROWS || AM == A_CONV)) {
      g.ksplit = ks;
      return launch_bn<128, AM, EM, 8, 512, 4, true>(g, b_i8, kpad, k, st);
    }
  }
#if B2_BYTES_BN128
  // u8 rows need no widening: re-reading A per 128-column tile is cheap and
  // buys the double-buffered accumulator
  if constexpr (AM == A_BYTES) return launch_bn<128, AM, EM, 8, 128>(g, b_i8, kpad, k, st);
#endif
  if (g.N > 128) {
    // few tiles (small batch): 128-column tiles, 512-element stages — twice
    // the CTAs and a quarter of the per-stage hand-offs on the serial K walk
    if constexpr (AM == A_ROWS || AM == A_CONV) {
      const int64_t tiles256 = ((g.M + BM - 1) / BM) * ((g.N + 255) / 256);
      if (B2_SMALLM_TILES && tiles256 < B2_SMALLM_TILES && (AM != A_CONV || g.spw % 4 == 0))
        return launch_bn<128, AM, EM, 8, 512>(g, b_i8, kpad, k, st);
    }
    return launch_bn<256, AM, EM, 8, 128>(g, b_i8, kpad, k, st);
  }
  if constexpr (AM == A_BYTECONV) {
    return launch_bn<128, AM, EM, 4, 128, B2_NEPI_BYTECONV>(g, b_i8, kpad, k, st);
  } else if constexpr (AM == A_BYTES) {
    return launch_bn<128, AM, EM, 8, 128>(g, b_i8, kpad, k, st);
  } else {
    if (AM == A_CONV && g.spw % 4 != 0) return launch_bn<128, AM, EM, 8, 128>(g, b_i8, kpad, k, st);
    return launch_bn<128, AM, EM, B2_NPW128, B2_BKS128>(g, b_i8, kpad, k, st);
  }
  }
}

inline int64_t kpad_of(int64_t k) { return (k + KPAD - 1) / KPAD * KPAD; }
constexpr int KPAD_F4 = 1024;  // fp4 weight rows: a multiple of the widest stage (512-byte rows)
inline int64_t kpad_f4(int64_t k) { return (k + KPAD_F4 - 1) / KPAD_F4 * KPAD_F4; }
template <bool F4>
inline int64_t kpad_for(int64_t k) { return F4 ? kpad_f4(k) : kpad_of(k); }
static_assert(KPAD % 128 == 0, "weight rows pad to whole TMA boxes");

inline bool conv_ok(int64_t batch, int h, int w, int c, int64_t filters, int kh, int kw, int stride, int pad) {
  if (!(batch >= 0 && h >= 1 && w >= 1 && c >= 1 && filters >= 1 && filters <= INT32_MAX && kh >= 1 && kw >= 1 &&
        stride >= 1 && pad >= 0 && h + 2 * pad >= kh && w + 2 * pad >= kw))
    return false;
  // output rows (and pool-window rows) are indexed in 32 bits on the device
  const int64_t ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  return batch * ho * wo < ((int64_t)1 << 31);
}

inline void conv_args(Args& g, const void* x, int64_t batch, int h, int w, int c, int kh, int kw, int stride,
                      int pad) {
  g.a = reinterpret_cast<const uint32_t*>(x);
  g.H = h;
  g.W = w;
  g.c = c;
  g.spw = c / 32;
  g.sstride = (int)(2 * wpl64(c));
  g.kh = kh;
  g.kw = kw;
  g.stride = stride;
  g.pad = pad;
  g.Ho = (h + 2 * pad - kh) / stride + 1;
  g.Wo = (w + 2 * pad - kw) / stride + 1;
  g.M = batch * g.Ho * g.Wo;
  // exact for dividends below 2^32 / divisor (K words and window cells here)
  g.spw_magic = ((1ull << 32) + (uint64_t)(g.spw > 0 ? g.spw : 1) - 1) / (uint64_t)(g.spw > 0 ? g.spw : 1);
  g.kw_magic = ((1ull << 32) + (uint64_t)kw - 1) / (uint64_t)kw;
}

// Padded-row implicit GEMM (tc_padrow.cuh) for the fp4 conv: stride 1,
// same-size output, odd kh == kw with pad = (k - 1) / 2, c % 128 == 0,
// at most 128 filters, weights resident (K <= 1536).
#ifndef B2_PADROW
#define B2_PADROW 1
#endif
// Band slot stride: the 16 KB minimum, or the band's planes rounded up to 1 KB.
inline int padrow_band_bytes(int64_t r8, int64_t planes) {
  const int64_t need = (r8 * 16 * planes + 1023) / 1024 * 1024;
  return (int)(need > PR_BAND_MAX ? need : PR_BAND_MAX);
}

// Shared padded-row geometry (virtual grid W + pad wide, H + pad tall per image).
inline void padrow_geometry(PadArgs& p, int64_t batch, int h, int w, int kh, int kw, int pad) {
  p.N = (int)batch;
  p.H = h;
  p.W = w;
  p.kh = kh;
  p.kw = kw;
  p.pad = pad;
  // pad zero columns per row and pad zero rows per image: a window reaching
  // pad cells past any edge lands on zeros
  p.Wp = w + (pad > 0 ? pad : 1);
  p.VI = (int64_t)(h + (pad > 0 ? pad : 1)) * p.Wp;
  p.Vtotal = p.VI * batch;
  // ceil(2^64 / VI) and ceil(2^32 / Wp): multiply-high division (vsplit) is
  // exact while v * ((-2^64) mod VI) < 2^64 and rem * ((-2^32) mod Wp) < 2^32
  // for every virtual row v and remainder rem < VI; padrow_exact checks the
  // sufficient bounds Vtotal * VI < 2^64 and VI * Wp < 2^32
  p.vi_magic = ~0ull / (uint64_t)p.VI + 1;
  p.wp_magic = (uint32_t)((((uint64_t)1 << 32) + p.Wp - 1) / p.Wp);
  p.band0 = pad * p.Wp + pad;  // the window's reach above (and below) a virtual row
  p.R8 = ((2 * p.band0 + BM) + 7) / 8 * 8;
}

inline bool padrow_exact(const PadArgs& p) {
  return (unsigned __int128)p.Vtotal * (unsigned __int128)p.VI < ((unsigned __int128)1 << 64) &&
         (uint64_t)p.VI * (uint64_t)p.Wp < ((uint64_t)1 << 32);
}

// Virtual-grid padded-row plan (packed-bit input): fills p with the
// geometry, band and weight shapes the launch uses and returns false when the
// layer does not qualify.  The path query (conv_path_f4) and the launch
// (padrow_launch -> padrow_run) both go through it, so eligibility and launch
// shape cannot drift apart.
inline bool padrow_plan(const Args& g, int c, int64_t filters, int64_t k, int64_t batch, PadArgs& p) {
  static const int on = [] {
    const char* e = getenv("B2_PADROW");
    return e ? atoi(e) : B2_PADROW;
  }();
  if (!on || g.stride != 1 || g.Ho != g.H || g.Wo != g.W || g.kh != g.kw || !(g.kh & 1) || g.pad != (g.kh - 1) / 2 ||
      c % 128 || filters > 256 || (filters <= 128 ? k > 1536 : k > 1280) || g.W >= 4096 || batch > INT32_MAX ||
      (int64_t)g.kh * g.kw * (c / 64) > 128 ||
      // enough tiles to fill the GPU (small batches keep the one-launch path)
      (int64_t)(g.H + 1) * (g.W + 1) * batch < (int64_t)BM * num_sms())
    return false;
  p = PadArgs{};
  padrow_geometry(p, batch, g.H, g.W, g.kh, g.kw, g.pad);
  if (!padrow_exact(p)) return false;  // e.g. a 4000 x 4000 1x1 conv: the index split would not be exact
  p.P = c / 32;
  p.nkb = (int)((k + 255) / 256);
  p.F = (int)filters;
  p.kmmas = p.P / 2;
  // the tile's band must fit the producer warps and one slot's 128 KB, and
  // the band ring shared memory next to the resident weights
  if ((int64_t)p.R8 * (p.P / 4) > 2 * 32 * PR_NPW || (int64_t)p.R8 * 16 * p.P > 128 * 1024) return false;
  p.band_bytes = padrow_band_bytes(p.R8, p.P);
  // threshold folded into one more MMA (tc_padrow.cuh BIAS): its K block may add an atom
  p.kk = (int)k;
  p.nkb_ld = p.nkb;
  if (B2_PR_VBIAS) {
    p.nkb = (int)((k + 64 + 255) / 256);
    if (k % 64) return false;
  }
  return (filters > 128 ? padrow_smem_bytes<256>(p.nkb, p.band_bytes, pr_bands<256>(), false, false, 0, B2_PR_VBIAS)
                        : padrow_smem_bytes<128>(p.nkb, p.band_bytes, pr_bands<128>(), false, false, 0, B2_PR_VBIAS)) <=
         227 * 1024;
}

// Row-aligned padded-row plan (tc_padrow.cuh ALIGN): tiles of 128 pixels
// covering whole rows of one image, kw column-shifted copies of the band,
// pooling fused into the epilogue.  Fills p (geometry, band ring, smem) and
// returns false when the layer does not qualify.  One routine decides
// eligibility and shapes the launch, so the two cannot drift apart.
#ifndef B2_PADROW_ALIGN
#define B2_PADROW_ALIGN 1
#endif
#ifndef B2_PADROW_PAIR
#define B2_PADROW_PAIR 0  // correct but measured slower; B2_PADROW_PAIR=1 opts in
#endif
inline bool padrow_align_plan(const Args& g, int c, int64_t filters, int64_t k, int64_t batch, int pool, PadArgs& p,
                              int& smem) {
  static const int on = [] {
    const char* e = getenv("B2_PADROW_ALIGN");
    return e ? atoi(e) : B2_PADROW_ALIGN;
  }();
  static const int min_bands = [] {
    const char* e = getenv("B2_ALIGN_MIN_BANDS");
    return e ? atoi(e) : 2;
  }();
  const int w = g.W, h = g.H;
  if (!on || g.stride != 1 || g.Ho != h || g.Wo != w || g.kh != g.kw || !(g.kh & 1) || g.pad != (g.kh - 1) / 2 ||
      c % 128 || filters > 256 || w < 1 || (w & (w - 1)) || BM % w || ((int64_t)h * w) % BM || batch > INT32_MAX)
    return false;
  const int tr = BM / w;  // image rows per tile
  if (pool && (tr & 1)) return false;
  if ((int64_t)g.kh * g.kw * (c / 64) > 128) return false;  // MMA offset table
  if (batch * h * w / BM < num_sms()) return false;          // too few tiles to fill the GPU
  p = PadArgs{};
  p.N = (int)batch;
  p.H = h;
  p.W = w;
  p.kh = g.kh;
  p.kw = g.kw;
  p.pad = g.pad;
  p.HW = (int64_t)h * w;
  p.wshift = 0;
  while ((1 << p.wshift) < w) ++p.wshift;
  p.Rb = (tr + 2 * g.pad) * w;
  p.R8 = (p.Rb + 7) / 8 * 8;
  p.P = c / 32;
  if ((int64_t)p.Rb * (p.P / 4) > 2 * 32 * PR_NPW) return false;  // band units per producer thread
  const int64_t band = ((int64_t)p.R8 * 16 * g.kw * p.P + 1023) / 1024 * 1024;
  if (band > 128 * 1024) return false;
  p.band_bytes = (int)band;
  p.nkb = (int)((k + 255) / 256);
  p.kmmas = p.P / 2;
  p.F = (int)filters;
  p.pool = pool;
  // CTA pairs (tc_padrow.cuh PAIR): half the weights per CTA, so a deeper band
  // ring fits; used when there are enough pair tiles for every SM pair
  static const int pair_env = [] {
    const char* e = getenv("B2_PADROW_PAIR");
    return e ? atoi(e) : B2_PADROW_PAIR;
  }();
  p.pair = pair_env && batch * h * w / BM >= 2 * (num_sms() / 2) ? 1 : 0;
  // filters on the MMA's M side with the weights in TMEM (tc_padrow.cuh TW):
  // <= 128 filters, K / 8 weight columns past PR_TW_COL, pooled rows <= 32 wide
  // (opt-in: with the loader warp the weights-in-shared-memory form is faster,
  // conv2 3.57 vs 3.94 ms — the per-lane ballot epilogue costs more issue
  // slots than the shared-memory bandwidth it saves)
  static const int tw_env = [] {
    const char* e = getenv("B2_PADROW_TW");
    return e ? atoi(e) : 0;
  }();
  p.tw = tw_env && !p.pair && filters <= 128 && PR_TW_COL + (k / 8 + 15) / 16 * 16 <= 512 && (!pool || w <= 32) ? 1 : 0;
  // single-CTA weights-in-shared-memory kernels fold the threshold into one
  // more K = 64 MMA (tc_padrow.cuh BIAS): its block may need one more atom,
  // and the bias (|T| + 1 <= K + 1) must fit the two-block encoding.  The
  // preferred shape (staging ring + folded threshold) falls back to register-
  // prefetching producers, then to the threshold table, when the resident
  // weights leave no room (256 filters at K = 1152: 160 KB).
  static const int nobias_env = [] {  // B2_ALIGN_NOBIAS=1: keep the threshold in the epilogue (A/B runs)
    const char* e = getenv("B2_ALIGN_NOBIAS");
    return e ? atoi(e) : 0;
  }();
  const bool bias_ok = !p.tw && !p.pair && k <= 5760 && k % 64 == 0 && !nobias_env;
  const int nkb0 = p.nkb;
  const int raw = g.sstride % 4 ? 0 : (int)((int64_t)p.Rb * g.sstride * 4);  // bulk copies move whole 16-byte pixels
  for (int opt = 0; opt < 3; ++opt) {
    const bool use_raw = opt == 0 && raw > 0, bias = opt < 2 && bias_ok;
    p.raw = use_raw ? 1 : 0;
    p.kk = bias ? (int)k : 0;
    p.nkb_ld = nkb0;
    p.nkb = bias ? (int)((k + 64 + 255) / 256) : nkb0;
    for (p.nbands = PR_BANDS_MAX; p.nbands >= min_bands; --p.nbands) {
      const int rb = use_raw ? raw : 0;
      smem = filters > 128 ? padrow_smem_bytes<256>(p.nkb, p.band_bytes, p.nbands, pool != 0, p.pair, rb, bias)
             : p.tw        ? padrow_smem_bytes<128>(0, p.band_bytes, p.nbands, pool != 0, false, rb, false)
                           : padrow_smem_bytes<128>(p.nkb, p.band_bytes, p.nbands, pool != 0, p.pair, rb, bias);
      if (smem <= 227 * 1024) return true;
    }
  }
  return false;
}



// Launch the padded-row kernel (and, pooled — only the opt-in byte-input
// entry b2_tc4_byte_conv_padrow — the bit-pool pass on a stream-ordered
// scratch).  p.nkb, p.P, p.kmmas, p.F, p.thresh/ge set by the caller.
template <bool BYTEIN>
inline int padrow_run(PadArgs& p, const int8_t* w, int64_t b_row_bytes, int pool, uint64_t* out, cudaStream_t st) {
  if ((int64_t)p.R8 * 16 * p.P > 128 * 1024 || (int64_t)p.R8 * (BYTEIN ? 1 : p.P / 4) > 2 * 32 * PR_NPW ||
      p.N < 0 || !padrow_exact(p))
    return B2_EINVAL;
  p.band_bytes = padrow_band_bytes(p.R8, p.P);
  p.ldo32 = 2 * wpl64(p.F);
  const bool wide = p.F > 128;  // one 256-column tile
  if (BYTEIN && wide) return B2_EINVAL;
  CUtensorMap map;
  if (int rc = make_bmap(&map, w, p.F, b_row_bytes, wide ? 256 : 128)) return rc;
  const int smem = wide ? padrow_smem_bytes<256>(p.nkb, p.band_bytes, pr_bands<256>(), false, false, 0, !BYTEIN && B2_PR_VBIAS)
                        : padrow_smem_bytes<128>(p.nkb, p.band_bytes, pr_bands<128>(), false, false, 0, !BYTEIN && B2_PR_VBIAS);
  static const bool generic_only = getenv("B2_PR_GENERIC") && atoi(getenv("B2_PR_GENERIC"));  // test hook
  const bool k3 = !generic_only && p.kh == 3 && p.kmmas == (BYTEIN ? 1 : 2);  // the unrolled 3x3 issue loops
  void (*kern)(CUtensorMap, PadArgs);
  if constexpr (BYTEIN)
    kern = k3 ? k_padrow_conv<3, 1, 128, true> : k_padrow_conv<0, 0, 128, true>;
  else
    kern = wide ? (k3 ? k_padrow_conv<3, 2, 256> : k_padrow_conv<0, 0, 256>)
                : (k3 ? k_padrow_conv<3, 2, 128> : k_padrow_conv<0, 0, 128>);
  // the size depends on the layer (weight atoms): opt in to the whole 227 KB
  // once per kernel and device, so any later, larger layer fits too
  static std::atomic<uint64_t> attr[4];
  if (smem > 227 * 1024) return B2_EINVAL;
  smem_optin(kern, 227 * 1024, attr[(wide ? 2 : 0) + (k3 ? 1 : 0)]);
  const int64_t tiles = (p.Vtotal + BM - 1) / BM;
  const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
  void* scratch = nullptr;
  if (pool) {  // unpooled thresholded bits, then the 2x2 OR/AND combine
    // stream-ordered scratch (capturable into graphs); keep the device's
    // default pool from returning it to the OS between calls
    static std::atomic<uint64_t> pool_kept{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(pool_kept.load() & (1ull << (dev & 63)))) {
      cudaMemPool_t mp;
      if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pool_kept.fetch_or(1ull << (dev & 63));
    }
    if (cudaError_t e = cudaMallocAsync(&scratch, (size_t)p.N * p.H * p.W * p.ldo32 * 4, st)) return (int)e;
    p.out_bits = reinterpret_cast<uint32_t*>(scratch);
  } else {
    p.out_bits = reinterpret_cast<uint32_t*>(out);
  }
  launch_k(kern, grid, 32 * (4 + PR_NPW + (wide ? pr_nepi<256>() : pr_nepi<128>())), smem, st, map, p);
  int rc = launched();
  if (pool) {
    if (!rc) {
      const int64_t n = (int64_t)p.N * (p.H / 2) * (p.W / 2);  // pooled sites
      launch_k(k_pool_bits, (unsigned)cdiv(n, 256), 256, 0, st, (const uint32_t*)scratch, (int64_t)p.N, p.H, p.W,
               p.ldo32, p.ge, p.F, reinterpret_cast<uint32_t*>(out));
      rc = launched();
    }
    cudaFreeAsync(scratch, st);
  }
  return rc;
}

// Launch the row-aligned kernel planned by padrow_align_plan (pool fused).
inline int padrow_align_run(PadArgs& p, int smem, const void* lines, int sstride, const int8_t* w, int64_t b_row_bytes,
                            const b2_thresh& th, uint64_t* out, cudaStream_t st, int64_t ldo32 = 0) {
  p.x = reinterpret_cast<const uint32_t*>(lines);
  p.sstride = sstride;
  p.thresh = th.thresh;
  p.ge = th.ge_dir;
  p.ldo32 = ldo32 ? ldo32 : 2 * wpl64(p.F);
  p.out_bits = reinterpret_cast<uint32_t*>(out);
  const bool wide = p.F > 128;
  CUtensorMap map;
  if (int rc = make_bmap(&map, w, p.F, b_row_bytes, wide ? 256 : 128)) return rc;
  static const bool generic_only = getenv("B2_PR_GENERIC") && atoi(getenv("B2_PR_GENERIC"));  // test hook
  const bool k3 = !generic_only && p.kh == 3 && p.kmmas == 2;
  const int threads = 32 * (4 + PR_NPW + (wide ? pr_nepi<256, true>() : pr_nepi<128, true>()));
  const int64_t tiles = (int64_t)p.N * p.HW / BM;
  if (p.tw) {
    p.wt = reinterpret_cast<const uint32_t*>(w);
    p.wt_words = (int)((int64_t)p.kh * p.kw * p.P * 4);  // K / 8
    p.wt_stride = (int)(b_row_bytes / 4);
    void (*kern)(CUtensorMap, PadArgs) =
        k3 ? k_padrow_conv<3, 2, 128, false, true, false, true> : k_padrow_conv<0, 0, 128, false, true, false, true>;
    static std::atomic<uint64_t> attr3[2];
    smem_optin(kern, 227 * 1024, attr3[k3 ? 1 : 0]);
    const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    launch_k(kern, grid, 32 * (4 + PR_NPW + pr_nepi<128, true, true>()), smem, st, map, p);
    return launched();
  }
  if (p.pair) {
    // weights split over the pair: TMA boxes of BNT / 2 rows
    if (int rc = make_bmap(&map, w, p.F, b_row_bytes, wide ? 128 : 64)) return rc;
    void (*kern)(CUtensorMap, PadArgs) =
        wide ? (k3 ? k_padrow_conv<3, 2, 256, false, true, true> : k_padrow_conv<0, 0, 256, false, true, true>)
             : (k3 ? k_padrow_conv<3, 2, 128, false, true, true> : k_padrow_conv<0, 0, 128, false, true, true>);
    static std::atomic<uint64_t> attr2[4];
    smem_optin(kern, 227 * 1024, attr2[(wide ? 2 : 0) + (k3 ? 1 : 0)]);
    const int64_t ptiles = (tiles + 1) / 2;
    const int64_t pairs = ptiles < num_sms() / 2 ? ptiles : num_sms() / 2;
    launch_kc(2, kern, (unsigned)(2 * pairs), threads, smem, st, map, p);
    return launched();
  }
  void (*kern)(CUtensorMap, PadArgs) =
      wide ? (k3 ? k_padrow_conv<3, 2, 256, false, true> : k_padrow_conv<0, 0, 256, false, true>)
           : (k3 ? k_padrow_conv<3, 2, 128, false, true> : k_padrow_conv<0, 0, 128, false, true>);
  static std::atomic<uint64_t> attr[4];
  smem_optin(kern, 227 * 1024, attr[(wide ? 2 : 0) + (k3 ? 1 : 0)]);
  const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
  launch_k(kern, grid, threads, smem, st, map, p);
  return launched();
}

// launch the virtual-grid kernel planned by padrow_plan (unpooled: pooled
// layers never take it, see conv_path_f4)
inline int padrow_launch(PadArgs& p, const Args& g, const void* lines, const int8_t* w_f4, int64_t k, uint64_t* out,
                         cudaStream_t st) {
  p.x = reinterpret_cast<const uint32_t*>(lines);
  p.sstride = g.sstride;
  p.thresh = g.thresh;
  p.ge = g.ge;
  return padrow_run<false>(p, w_f4, kpad_f4(k) / 2, 0, out, st);
}

// Kernel choice of the fused fp4 conv (b2_tc4_conv_bn_pack), also exported
// as b2_tc4_conv_path so tests can assert which kernel a case exercised.
enum ConvPath { PATH_IM2COL = 0, PATH_SPLITK = 1, PATH_PADROW = 2, PATH_PADROW_ALIGNED = 3 };
inline bool align_split_on() {  // B2_ALIGN_SPLIT=0: 129-256 filters in one 256-column launch
  static const int on = [] {
    const char* e = getenv("B2_ALIGN_SPLIT");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}
inline int conv_path_f4(const Args& g, int c, int64_t filters, int64_t k, int64_t batch, int pool, PadArgs& p,
                        int& smem) {
  if (!batch) return PATH_IM2COL;
  if (splitk_count<A_CONV, E_PACK>(g, k)) return PATH_SPLITK;
  if (padrow_align_plan(g, c, filters, k, batch, pool, p, smem)) return PATH_PADROW_ALIGNED;
  // 129-256 filters whose 256-column form does not fit (pooled): two
  // 128-filter launches (conv_bn_pack splits every aligned layer this wide)
  if (filters > 128 && filters <= 256 && align_split_on() && padrow_align_plan(g, c, 128, k, batch, pool, p, smem))
    return PATH_PADROW_ALIGNED;
  // pooled layers the row-aligned kernel cannot take use the im2col kernel's
  // fused pool: the virtual grid's pool windows straddle tiles, and an
  // unpooled scratch would be an allocation inside the forward pass
  if (!pool && padrow_plan(g, c, filters, k, batch, p)) return PATH_PADROW;
  return PATH_IM2COL;
}

inline void pack_args(Args& g, const b2_thresh& th, uint64_t* out, int64_t n) {
  g.out_bits = reinterpret_cast<uint32_t*>(out);
  g.ldo32 = 2 * wpl64(n);
  g.thresh = th.thresh;
  g.ge = th.ge_dir;
}

template <bool F4>
int bgemm(const uint64_t* a, int64_t m, const int8_t* b_i8, int64_t n, int64_t wpl, int32_t k, int32_t* out,
                void* stream) {
  if (m < 0 || n < 0 || wpl < 1 || k < 1 || k > 64 * wpl || n > INT32_MAX) return B2_EINVAL;
  Args g{};
  g.a = reinterpret_cast<const uint32_t*>(a);
  g.lda = 2 * wpl;
  g.awords = (k + 31) / 32;
  g.M = m;
  g.N = (int)n;
  g.out_i32 = out;
  g.ldo = n;
  return launch<A_ROWS, E_I32, F4>(g, b_i8, kpad_for<F4>(k), S(stream), k);
}

template <bool F4>
int dense_affine_f64(const uint64_t* x, int64_t batch, const int8_t* w_i8, int64_t units, int64_t wpl,
                           int32_t k, const double* mean, const double* scale, const double* beta, double* out,
                           void* stream) {
  if (units < 1 || units > INT32_MAX || batch < 0 || wpl < 1 || k < 1 || k > 64 * wpl || !mean || !scale || !beta)
    return B2_EINVAL;
  Args g{};
  g.a = reinterpret_cast<const uint32_t*>(x);
  g.lda = 2 * wpl;
  g.awords = (k + 31) / 32;
  g.M = batch;
  g.N = (int)units;
  g.mean = mean;
  g.scale = scale;
  g.beta = beta;
  g.out_f64 = out;
  g.ldo = units;
  return launch<A_ROWS, E_AFFINE, F4>(g, w_i8, kpad_for<F4>(k), S(stream), k);
}

template <bool F4>
int dense_bn_pack(const uint64_t* x, int64_t batch, const int8_t* w_i8, int64_t units, int64_t wpl, int32_t k,
                        b2_thresh th, uint64_t* out, void* stream) {
  if (units < 1 || units > INT32_MAX || batch < 0 || wpl < 1 || k < 1 || k > 64 * wpl || !th.thresh || !th.ge_dir)
    return B2_EINVAL;
  Args g{};
  g.a = reinterpret_cast<const uint32_t*>(x);
  g.lda = 2 * wpl;
  g.awords = (k + 31) / 32;
  g.M = batch;
  g.N = (int)units;
  pack_args(g, th, out, units);
  return launch<A_ROWS, E_PACK, F4>(g, w_i8, kpad_for<F4>(k), S(stream), k);
}

template <bool F4>
int conv_forward(const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* w_i8,
                       int64_t filters, int kh, int kw, int stride, int pad, int32_t* out, void* stream) {
  if (!conv_ok(batch, h, w, c, filters, kh, kw, stride, pad) || c % 64) return B2_EINVAL;
  Args g{};
  conv_args(g, lines, batch, h, w, c, kh, kw, stride, pad);
  const int64_t k = (int64_t)kh * kw * c;
  g.N = (int)filters;
  g.out_i32 = out;
  g.ldo = filters;
  return launch<A_CONV, E_I32, F4>(g, w_i8, kpad_for<F4>(k), S(stream), k);
}

template <bool F4>
int conv_bn_pack(const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* w_i8,
                       int64_t filters, int kh, int kw, int stride, int pad, int pool, b2_thresh th, uint64_t* out,
                       void* stream) {
  if (!conv_ok(batch, h, w, c, filters, kh, kw, stride, pad) || c % 64 || !th.thresh || !th.ge_dir)
    return B2_EINVAL;
  Args g{};
  conv_args(g, lines, batch, h, w, c, kh, kw, stride, pad);
  if (pool && ((g.Ho & 1) || (g.Wo & 1))) return B2_EINVAL;
  const int64_t k = (int64_t)kh * kw * c;
  g.N = (int)filters;
  pack_args(g, th, out, filters);
  if constexpr (F4) {
    PadArgs p;
    int smem = 0;
    switch (conv_path_f4(g, c, filters, k, batch, pool, p, smem)) {
      case PATH_PADROW_ALIGNED: {
        // 129-256 filters: two launches of the 128-filter kernel (each its
        // own 64 of the output's 128-bit words per 128 filters) — triple-
        // buffered 128-column accumulators instead of one 256-column
        // accumulator whose drain the MMA thread waited on 29 % of the time
        PadArgs p2;
        int smem2 = 0;
        if (filters > 128 && align_split_on() && padrow_align_plan(g, c, 128, k, batch, pool, p2, smem2)) {
          const int64_t ldo32 = 2 * wpl64(filters);
          for (int part = 0; part < 2; ++part) {
            PadArgs ph = p2;
            ph.F = part ? (int)(filters - 128) : 128;
            ph.wlim = (int)(part ? ldo32 - 4 : 4);  // this part's 32-bit words of each pixel
            b2_thresh th2 = th;
            th2.thresh += 128 * part;
            th2.ge_dir += 128 * part;
            if (th2.thresh64) th2.thresh64 += 128 * part;
            if (int rc = padrow_align_run(ph, smem2, lines, g.sstride, w_i8 + 128 * part * (kpad_f4(k) / 2), kpad_f4(k) / 2,
                                          th2, out + 2 * part, S(stream), ldo32))
              return rc;
          }
          return 0;
        }
        return padrow_align_run(p, smem, lines, g.sstride, w_i8, kpad_f4(k) / 2, th, out, S(stream));
      }
      case PATH_PADROW: return padrow_launch(p, g, lines, w_i8, k, out, S(stream));
      default: break;
    }
  }
  if (pool) return launch<A_CONV, E_POOLPACK, F4>(g, w_i8, kpad_for<F4>(k), S(stream), k);
  return launch<A_CONV, E_PACK, F4>(g, w_i8, kpad_for<F4>(k), S(stream), k);
}

// Fused first layer (tc_byteconv.cuh): row-aligned tiles, window K <= 31
// bits (+ the folded threshold) in one int8 MMA, no unrolled scratch.
#ifndef B2_BYTECONV_FUSED
#define B2_BYTECONV_FUSED 1
#endif
inline bool byteconv_fused_ok(int64_t batch, int h, int w, int c, int64_t filters, int kh, int kw, int stride, int pad,
                              int pool) {
  static const int on = [] {
    const char* e = getenv("B2_BYTECONV_FUSED");
    return e ? atoi(e) : B2_BYTECONV_FUSED;
  }();
  if (!on || pool || stride != 1 || kh != kw || !(kh & 1) || pad != (kh - 1) / 2 || c < 1 || c > 3 ||
      (int64_t)kh * kw * c > 31 || filters < 1 || filters > 256 || w < 1 || (w & (w - 1)) || BM % w ||
      ((int64_t)h * w) % BM || batch < 1 || batch * h * w >= ((int64_t)1 << 31))
    return false;
  // the tile's code band, and its raw rows as one TMA box (row pitch a multiple
  // of 16 bytes, at most 256 bytes wide)
  const int64_t rowb = (int64_t)w * c, brows = BM / w + 2 * pad;
  return brows * w <= 1024 && rowb % 16 == 0 && rowb <= 256 && brows <= 256 && brows * rowb <= BC_RAW_BYTES;
}

inline int byteconv_fused_run(const uint8_t* x, int64_t batch, int h, int w, int c, const b2_thresh& th_in,
                              const int8_t* w_i8, int64_t filters, int kh, int kw, int pad, const b2_thresh& th_out,
                              uint64_t* out, cudaStream_t st) {
  ByteConvArgs g{};
  g.x = x;
  g.N = (int)batch;
  g.H = h;
  g.W = w;
  g.c = c;
  g.kh = kh;
  g.kw = kw;
  g.pad = pad;
  g.HW = (int64_t)h * w;
  g.tpi = (uint32_t)(g.HW / BM);
  while ((1 << g.wshift) < w) ++g.wshift;
  g.K = kh * kw * c;
  g.th_in = th_in.thresh;
  g.ge_in = th_in.ge_dir;
  g.w = w_i8;
  g.wpitch = kpad_of(g.K);
  g.F = (int)filters;
  g.thresh = th_out.thresh;
  g.ge = th_out.ge_dir;
  g.out_bits = reinterpret_cast<uint32_t*>(out);
  g.ldo32 = 2 * wpl64(filters);
  // the image as (N*H rows) x (W*c bytes) for the producers' band TMA
  auto fn = encode_fn();
  if (!fn) return B2_EINVAL;
  CUtensorMap xmap;
  cuuint64_t dims[2] = {(cuuint64_t)w * c, (cuuint64_t)batch * h};
  cuuint64_t strides[1] = {(cuuint64_t)w * c};
  cuuint32_t box[2] = {(cuuint32_t)(w * c), (cuuint32_t)(BM / w + 2 * pad)};
  cuuint32_t estr[2] = {1, 1};
  if (fn(&xmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(x), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return B2_EINVAL;
  const bool wide = filters > 128, k3 = kh == 3 && w <= 32;  // row triples by shuffle: a row within one warp
  // the 3x3 / 3-channel first layer (RGB images) with compile-time channels
  void (*kern)(CUtensorMap, ByteConvArgs) =
      wide ? (k3 ? (c == 3 ? k_byteconv<256, 3, 3> : k_byteconv<256, 3>) : k_byteconv<256, 0>)
           : (k3 ? (c == 3 ? k_byteconv<128, 3, 3> : k_byteconv<128, 3>) : k_byteconv<128, 0>);
  const int smem = wide ? bc_smem_bytes<256>() : bc_smem_bytes<128>();
  static std::atomic<uint64_t> attr[6];
  smem_optin(kern, smem, attr[(wide ? 3 : 0) + (k3 ? (c == 3 ? 2 : 1) : 0)]);
  const int64_t tiles = batch * g.HW / BM;
  const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
  launch_k(kern, grid, 32 * (4 + BC_NPW + BC_NEPI), smem, st, xmap, g);
  return launched();
}

template <bool F4>
int byte_conv_bn_pack(const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in,
                            const int8_t* w_i8, int64_t filters, int kh, int kw, int stride, int pad, int pool,
                            b2_thresh th_out, void* scratch, uint64_t* out, void* stream) {
  if (!conv_ok(batch, h, w, c, filters, kh, kw, stride, pad) || (int64_t)kh * kw * c > BK || c > 8 || !scratch ||
      !th_in.thresh || !th_in.ge_dir || !th_out.thresh || !th_out.ge_dir)
    return B2_EINVAL;
  Args g{};
  conv_args(g, x, batch, h, w, c, kh, kw, stride, pad);
  if (pool && ((g.Ho & 1) || (g.Wo & 1))) return B2_EINVAL;
  if (!batch) return 0;
  if (!F4 && byteconv_fused_ok(batch, h, w, c, filters, kh, kw, stride, pad, pool))
    return byteconv_fused_run(x, batch, h, w, c, th_in, w_i8, filters, kh, kw, pad, th_out, out, S(stream));
  const int64_t k = (int64_t)kh * kw * c;
  const int kw32 = (int)((k + 31) / 32);
  {
    int band = batch * ((g.Ho + BAND - 1) / BAND) >= 2 * num_sms() ? BAND : BAND_SMALL;
    if ((size_t)((band - 1) * stride + kh) * w > 48 * 1024) band = BAND_SMALL;  // wide images: small bands
    const int bands = (g.Ho + band - 1) / band;
    const int in_rows = (band - 1) * stride + kh;
    const size_t smem = (size_t)in_rows * w;
    if (smem > 48 * 1024 || batch * bands > INT32_MAX) return B2_EINVAL;
    auto kern = (kh == 3 && kw == 3 && c == 3) ? k_byte_unroll<3, 3, 3> : k_byte_unroll<0, 0, 0>;
    launch_k(kern, (unsigned)(batch * bands), 256, smem, S(stream), x, h, w, c, kh, kw, stride, pad, g.Ho, g.Wo,
             kw32, pool, band, th_in.thresh, th_in.ge_dir, reinterpret_cast<uint32_t*>(scratch));
  }
  if (int rc = launched()) return rc;
  // rows are ordered like the conv output (pool-window-major when pooled)
  g.a = reinterpret_cast<const uint32_t*>(scratch);
  g.lda = 2 * kw32;
  g.awords = kw32;
  g.N = (int)filters;
  g.nkb = 1;
  pack_args(g, th_out, out, filters);
  if (pool) return launch<A_BYTECONV, E_POOLPACK, F4>(g, w_i8, kpad_for<F4>(k), S(stream), k);
  return launch<A_BYTECONV, E_PACK, F4>(g, w_i8, kpad_for<F4>(k), S(stream), k);
}

}  // namespace tc
}  // namespace b2

using namespace b2;

extern "C" {

int64_t b2_i8_kpad(int64_t k) { return tc::kpad_of(k); }

int b2_expand_i8(const uint64_t* w, int64_t rows, int64_t wpl, int64_t k, int permute, int8_t* out, void* stream) {
  if (rows < 0 || wpl < 1 || k < 1 || k > 64 * wpl) return B2_EINVAL;
  int64_t kpad = tc::kpad_of(k);
  int64_t n = rows * kpad / 4;
  if (!n) return 0;
  launch_k(tc::k_expand_i8, (unsigned)cdiv(n, 256), 256, 0, S(stream), w, rows, wpl, k, kpad, permute, out);
  return launched();
}

int64_t b2_f4_kpad(int64_t k) { return tc::kpad_f4(k); }

int64_t b2_f4_cells_row_bytes(int cells) { return cells < 1 ? -1 : tc::kpad_f4((int64_t)cells * 64) / 2; }

int b2_expand_f4_cells(const uint64_t* w, int64_t rows, int64_t wpl, int cells, int c, uint8_t* out, void* stream) {
  if (rows < 0 || cells < 1 || c < 1 || c > 8 || (int64_t)cells * c > 64 * wpl) return B2_EINVAL;
  const int64_t row_words = tc::kpad_f4((int64_t)cells * 64) / 8;
  const int64_t n = rows * row_words;
  if (!n) return 0;
  launch_k(tc::k_expand_f4_cells, (unsigned)cdiv(n, 256), 256, 0, S(stream), w, rows, wpl, cells, c, row_words,
           reinterpret_cast<uint32_t*>(out));
  return launched();
}

int b2_tc4_byte_conv_padrow(const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in,
                            const uint8_t* w_cells, int64_t filters, int kh, int kw, int pad, int pool,
                            b2_thresh th_out, uint64_t* out, void* stream) {
  if (!tc::conv_ok(batch, h, w, c, filters, kh, kw, 1, pad) || c > 8 || filters > 128 || kh != kw || !(kh & 1) ||
      pad != (kh - 1) / 2 || kh * kw > 128 || !th_in.thresh || !th_in.ge_dir || !th_out.thresh || !th_out.ge_dir ||
      (pool && ((h & 1) || (w & 1))) || batch > INT32_MAX || w >= 4096)
    return B2_EINVAL;
  if (!batch) return 0;
  tc::PadArgs p{};
  tc::padrow_geometry(p, batch, h, w, kh, kw, pad);
  p.xb = x;
  p.cin = c;
  p.th_in = th_in.thresh;
  p.ge_in = th_in.ge_dir;
  p.P = 2;  // data plane + zero plane: one K=64 MMA per window cell
  p.kmmas = 1;
  p.nkb = (int)((kh * kw * 64 + 255) / 256);
  p.F = (int)filters;
  p.thresh = th_out.thresh;
  p.ge = th_out.ge_dir;
  return tc::padrow_run<true>(p, reinterpret_cast<const int8_t*>(w_cells), b2_f4_cells_row_bytes(kh * kw), pool, out,
                              S(stream));
}

int b2_expand_f4(const uint64_t* w, int64_t rows, int64_t wpl, int64_t k, uint8_t* out, void* stream) {
  if (rows < 0 || wpl < 1 || k < 1 || k > 64 * wpl) return B2_EINVAL;
  const int64_t kpad = tc::kpad_f4(k);
  const int64_t n = rows * kpad / 8;
  if (!n) return 0;
  launch_k(tc::k_expand_f4, (unsigned)cdiv(n, 256), 256, 0, S(stream), w, rows, wpl, k, kpad,
           reinterpret_cast<uint32_t*>(out));
  return launched();
}

#define B2_TC_WRAP(NAME, IMPL, PARAMS, ARGS)                              \
  int b2_tc_##NAME PARAMS { return tc::IMPL<false> ARGS; }                \
  int b2_tc4_##NAME PARAMS { return tc::IMPL<true> ARGS; }

B2_TC_WRAP(bgemm, bgemm,
           (const uint64_t* a, int64_t m, const int8_t* b, int64_t n, int64_t wpl, int32_t k, int32_t* out,
            void* stream),
           (a, m, b, n, wpl, k, out, stream))
B2_TC_WRAP(dense_affine_f64, dense_affine_f64,
           (const uint64_t* x, int64_t batch, const int8_t* w, int64_t units, int64_t wpl, int32_t k,
            const double* mean, const double* scale, const double* beta, double* out, void* stream),
           (x, batch, w, units, wpl, k, mean, scale, beta, out, stream))
B2_TC_WRAP(dense_bn_pack, dense_bn_pack,
           (const uint64_t* x, int64_t batch, const int8_t* w, int64_t units, int64_t wpl, int32_t k, b2_thresh th,
            uint64_t* out, void* stream),
           (x, batch, w, units, wpl, k, th, out, stream))
B2_TC_WRAP(conv_forward, conv_forward,
           (const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* wt, int64_t filters, int kh,
            int kw, int stride, int pad, int32_t* out, void* stream),
           (lines, batch, h, w, c, wt, filters, kh, kw, stride, pad, out, stream))
B2_TC_WRAP(conv_bn_pack, conv_bn_pack,
           (const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* wt, int64_t filters, int kh,
            int kw, int stride, int pad, int pool, b2_thresh th, uint64_t* out, void* stream),
           (lines, batch, h, w, c, wt, filters, kh, kw, stride, pad, pool, th, out, stream))
B2_TC_WRAP(byte_conv_bn_pack, byte_conv_bn_pack,
           (const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in, const int8_t* wt,
            int64_t filters, int kh, int kw, int stride, int pad, int pool, b2_thresh th_out, void* scratch,
            uint64_t* out, void* stream),
           (x, batch, h, w, c, th_in, wt, filters, kh, kw, stride, pad, pool, th_out, scratch, out, stream))
#undef B2_TC_WRAP

int b2_tc_input8_bn_pack(const uint8_t* x, int64_t batch, int64_t k, const int8_t* w_i8, int64_t units, b2_thresh th,
                         uint64_t* out, void* stream) {
  if (batch < 0 || k < 1 || k % 4 || units < 1 || units > INT32_MAX || !th.thresh || !th.ge_dir) return B2_EINVAL;
  tc::Args g{};
  g.a = reinterpret_cast<const uint32_t*>(x);
  g.lda = k / 4;
  g.awords = (int)(k / 4);
  g.M = batch;
  g.N = (int)units;
  tc::pack_args(g, th, out, units);
  // u8 rows whose pitch and base TMA can address: loaded by TMA straight into
  // shared memory (no producer warps), int8 MMA with A from shared memory
  static const int use_tma = [] {
    const char* e = getenv("B2_INPUT8_TMA");
    return e ? atoi(e) : 1;
  }();
  if (use_tma && batch && k % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && batch <= INT32_MAX) {
    auto fn = tc::encode_fn();
    CUtensorMap amap;
    cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)batch};
    cuuint64_t strides[1] = {(cuuint64_t)k};
    cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)tc::BM};
    cuuint32_t estr[2] = {1, 1};
    if (fn && fn(&amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(x), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      return tc::launch<tc::A_BYTES_TMA, tc::E_PACK>(g, w_i8, tc::kpad_of(k), S(stream), k, &amap);
  }
  return tc::launch<tc::A_BYTES, tc::E_PACK>(g, w_i8, tc::kpad_of(k), S(stream), k);
}

int b2_tc4_conv_path(int64_t batch, int h, int w, int c, int64_t filters, int kh, int kw, int stride, int pad,
                     int pool) {
  if (!tc::conv_ok(batch, h, w, c, filters, kh, kw, stride, pad) || c % 64) return -1;
  tc::Args g{};
  tc::conv_args(g, nullptr, batch, h, w, c, kh, kw, stride, pad);
  g.N = (int)filters;
  tc::PadArgs p;
  int smem = 0;
  return tc::conv_path_f4(g, c, filters, (int64_t)kh * kw * c, batch, pool, p, smem);
}

int b2_tc_byte_conv_path(int64_t batch, int h, int w, int c, int64_t filters, int kh, int kw, int stride, int pad,
                         int pool) {
  if (!tc::conv_ok(batch, h, w, c, filters, kh, kw, stride, pad) || c > 8 || (int64_t)kh * kw * c > tc::BK) return -1;
  return tc::byteconv_fused_ok(batch, h, w, c, filters, kh, kw, stride, pad, pool) ? 1 : 0;
}

int64_t b2_tc_byte_conv_scratch_bytes(int64_t batch, int h, int w, int c, int kh, int kw, int stride, int pad) {
  if (!tc::conv_ok(batch, h, w, c, 1, kh, kw, stride, pad)) return -1;
  const int64_t ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  const int64_t kw32 = ((int64_t)kh * kw * c + 31) / 32;
  return batch * ho * wo * 2 * kw32 * 4;
}

}  // extern "C"
