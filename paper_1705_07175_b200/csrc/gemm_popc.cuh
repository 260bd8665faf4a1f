// Tiled XOR-popcount GEMM for sm_100a (LOP3 + POPC on the CUDA cores).
//
//   acc[m, n] = popc(A_m XOR B_n) summed over the K words,
//   dot[m, n] = K - 2 * acc                        (_kernels.py:85-106)
//
// A rows come either from a plain row-major packed matrix or from an
// IMPLICIT bit-im2col gather of a batched NHWC-bits activation tensor
// (_kernels.py:170-199 without materialising the unrolled matrix: when
// C % 32 == 0 every window cell is a run of whole uint32 words, so the
// unrolled row is a concatenation of site words and out-of-bounds sites
// are zero-filled by cp.async).  B rows are the filters / weight rows.
//
// CTA: 256 threads = WARPS_M x WARPS_N warps; a warp owns TM rows and
// 32*TN columns, lane l holding columns l, l+32, ... so that the 32 lanes
// of one column group produce one packed output word with __ballot_sync
// (channel-fastest packing, bit i = channel 32*j + i).  3-stage cp.async
// pipeline, BK = 32 words (1024 bits) per stage; A fragments are smem
// broadcasts, B fragments are conflict-free LDS.128 (row pitch 36 words).
//
// Epilogues (MODE):
//   EPI_I32      int32 dot (+ padding correction)      conv_forward / bgemm
//   EPI_PACK     threshold + sign + ballot repack      _PackedBN after conv/dense
//   EPI_POOLPACK 2x2 max over the 4 rows of a pool window, then EPI_PACK
//                (rows are ordered pool-window-major, see conv_row())
#pragma once
#include "common.cuh"

namespace b2 {

enum { EPI_I32 = 0, EPI_PACK = 1, EPI_POOLPACK = 2 };

struct GemmArgs {
  // A: plain rows
  const uint32_t* a;
  int64_t lda;  // uint32 words per A row
  // A: implicit conv gather (batched NHWC-bits input)
  int H, W, spw, sstride;  // spw = used uint32 words per site (C/32), sstride = site pitch in words
  int kw_, stride, pad, Ho, Wo;
  // B
  const uint32_t* b;
  int64_t ldb;
  int kwords;  // uint32 words of K to process (A and B)
  int64_t M;
  int N;
  int32_t kbits;
  // epilogue
  const int32_t* corr;  // (Ho*Wo, N) or null
  int32_t* out_i32;
  int64_t ldo;
  uint32_t* out_bits;
  int64_t ldo32;  // uint32 words per output line
  const int32_t* thresh;
  const uint8_t* ge;
};

template <int WARPS_M, int WARPS_N, int TM, int TN>
struct TileCfg {
  static constexpr int BM = WARPS_M * TM;
  static constexpr int BN = WARPS_N * 32 * TN;
  static constexpr int BK = 32;
  static constexpr int LDS = BK + 4;
  static constexpr int STAGES = 3;
  static constexpr int SMEM = STAGES * (BM + BN) * LDS * 4;
};

// Output row -> (image, oy, ox).  Pool-ordered rows group each 2x2 window's
// four positions in consecutive rows: m = 4*q + 2*cy + cx.
template <bool POOLED>
__device__ __forceinline__ void conv_row(const GemmArgs& g, int64_t m, int64_t& img, int& oy, int& ox) {
  if constexpr (POOLED) {
    int64_t q = m >> 2;
    int cell = (int)(m & 3);
    int hp = g.Ho >> 1, wp = g.Wo >> 1;
    img = q / (hp * wp);
    int r = (int)(q - img * (hp * wp));
    oy = 2 * (r / wp) + (cell >> 1);
    ox = 2 * (r % wp) + (cell & 1);
  } else {
    int64_t hw = (int64_t)g.Ho * g.Wo;
    img = m / hw;
    int r = (int)(m - img * hw);
    oy = r / g.Wo;
    ox = r % g.Wo;
  }
}

template <class Cfg, int CWA, int CWB, bool CONV, int MODE, int TM, int TN, int WARPS_N>
__global__ void __launch_bounds__(256, 2) k_popc_gemm(const GemmArgs g) {
  pdl_entry();
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, LDS = Cfg::LDS, STAGES = Cfg::STAGES;
  constexpr int A_CPR = BK / CWA;  // A chunks per row per stage
  constexpr int A_CHUNKS = BM * A_CPR / 256;
  constexpr int B_CPR = BK / CWB;
  constexpr int B_CHUNKS = BN * B_CPR / 256;
  static_assert(BM * A_CPR % 256 == 0 && BN * B_CPR % 256 == 0, "chunking");
  constexpr bool POOLED = (MODE == EPI_POOLPACK);

  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* As = smem;
  uint32_t* Bs = smem + STAGES * BM * LDS;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int warp_m = warp / WARPS_N, warp_n = warp % WARPS_N;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;

  // per-thread A chunk geometry (fixed across K tiles)
  const uint32_t* a_base[A_CHUNKS];
  int a_iy[A_CHUNKS], a_ix[A_CHUNKS];
  bool a_ok[A_CHUNKS];
#pragma unroll
  for (int i = 0; i < A_CHUNKS; ++i) {
    int idx = tid + i * 256;
    int64_t m = m0 + idx / A_CPR;
    a_ok[i] = m < g.M;
    if constexpr (CONV) {
      int64_t img = 0;
      int oy = 0, ox = 0;
      if (a_ok[i]) conv_row<POOLED>(g, m, img, oy, ox);
      a_base[i] = g.a + img * (int64_t)g.H * g.W * g.sstride;
      a_iy[i] = oy * g.stride - g.pad;
      a_ix[i] = ox * g.stride - g.pad;
    } else {
      a_base[i] = g.a + (a_ok[i] ? m : 0) * g.lda;
      a_iy[i] = a_ix[i] = 0;
    }
  }

  auto load_tile = [&](int kt, int stage) {
    const int k0 = kt * BK;
    uint32_t* as = As + stage * BM * LDS;
    uint32_t* bs = Bs + stage * BN * LDS;
#pragma unroll
    for (int i = 0; i < A_CHUNKS; ++i) {
      int idx = tid + i * 256;
      int r = idx / A_CPR, kc = idx % A_CPR;
      int kw = k0 + kc * CWA;
      bool ok = a_ok[i] && kw < g.kwords;
      const uint32_t* src = g.a;
      if constexpr (CONV) {
        int cell = kw / g.spw;
        int within = kw - cell * g.spw;
        int dy = cell / g.kw_, dx = cell - dy * g.kw_;
        int iy = a_iy[i] + dy, ix = a_ix[i] + dx;
        ok = ok && iy >= 0 && iy < g.H && ix >= 0 && ix < g.W;
        if (ok) src = a_base[i] + ((int64_t)iy * g.W + ix) * g.sstride + within;
      } else {
        if (ok) src = a_base[i] + kw;
      }
      cp_async_zfill<CWA * 4>(as + r * LDS + kc * CWA, src, ok);
    }
#pragma unroll
    for (int i = 0; i < B_CHUNKS; ++i) {
      int idx = tid + i * 256;
      int r = idx / B_CPR, kc = idx % B_CPR;
      int kw = k0 + kc * CWB;
      int n = n0 + r;
      bool ok = n < g.N && kw < g.kwords;
      const uint32_t* src = ok ? g.b + (int64_t)n * g.ldb + kw : g.b;
      cp_async_zfill<CWB * 4>(bs + r * LDS + kc * CWB, src, ok);
    }
  };

  uint32_t acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0;

  const int ktiles = (g.kwords + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < ktiles) load_tile(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
    cp_async_commit();
    const uint32_t* as = As + (kt % STAGES) * BM * LDS + (warp_m * TM) * LDS;
    const uint32_t* bs = Bs + (kt % STAGES) * BN * LDS + (warp_n * 32 * TN + lane) * LDS;
    const int kend = g.kwords - kt * BK;  // the last tile may be partial (e.g. K = 36 words)
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if (kk >= kend) break;  // warp-uniform
      uint4 bv[TN];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = *reinterpret_cast<const uint4*>(bs + j * 32 * LDS + kk);
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        uint4 av = *reinterpret_cast<const uint4*>(as + i * LDS + kk);
#pragma unroll
        for (int j = 0; j < TN; ++j)
          acc[i][j] += __popc(av.x ^ bv[j].x) + __popc(av.y ^ bv[j].y) + __popc(av.z ^ bv[j].z) +
                       __popc(av.w ^ bv[j].w);
      }
    }
  }
  cp_async_wait<0>();

  // ---------------------------------------------------------------- epilogue
  const int64_t mw = m0 + warp_m * TM;
  const int nw = n0 + warp_n * 32 * TN;
  if constexpr (MODE == EPI_I32) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      int64_t m = mw + i;
      if (m >= g.M) continue;
      int pos = 0;
      if constexpr (CONV) pos = (int)(m % ((int64_t)g.Ho * g.Wo));
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        int n = nw + 32 * j + lane;
        if (n < g.N) {
          int32_t v = g.kbits - 2 * (int32_t)acc[i][j];
          if (g.corr) v += g.corr[(int64_t)pos * g.N + n];
          g.out_i32[m * g.ldo + n] = v;
        }
      }
    }
  } else {
    int32_t t[TN];
    bool ge[TN], nok[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int n = nw + 32 * j + lane;
      nok[j] = n < g.N;
      t[j] = nok[j] ? g.thresh[n] : 0;
      ge[j] = nok[j] ? g.ge[n] != 0 : true;
    }
    constexpr int G = POOLED ? 4 : 1;  // rows per output site
#pragma unroll
    for (int s = 0; s < TM / G; ++s) {
      int64_t mrow = mw + s * G;
      bool mok = mrow < g.M;  // pool groups are whole (M % 4 == 0)
      int pos[G];
#pragma unroll
      for (int r = 0; r < G; ++r) {
        pos[r] = 0;
        if constexpr (CONV) {
          if (mok && g.corr) {
            int64_t img;
            int oy, ox;
            conv_row<POOLED>(g, mrow + r, img, oy, ox);
            pos[r] = oy * g.Wo + ox;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        int n = nw + 32 * j + lane;
        int32_t v = INT32_MIN;
#pragma unroll
        for (int r = 0; r < G; ++r) {
          int32_t d = g.kbits - 2 * (int32_t)acc[s * G + r][j];
          if (CONV && g.corr && mok && nok[j]) d += g.corr[(int64_t)pos[r] * g.N + n];
          v = d > v ? d : v;
        }
        bool bit = mok && nok[j] && thr_bit(v, t[j], ge[j]);
        uint32_t word = __ballot_sync(0xffffffffu, bit);
        int64_t widx = (nw + 32 * j) >> 5;
        if (mok && widx < g.ldo32 && lane == ((s * TN + j) & 31)) g.out_bits[(mrow / G) * g.ldo32 + widx] = word;
      }
    }
  }
}

}  // namespace b2
