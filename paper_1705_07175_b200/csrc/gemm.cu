// Binary GEMM / conv entry points (SURVEY.md §8 a-6 .. a-10).
#include "gemm_popc.cuh"

namespace b2 {

using Cfg = TileCfg<4, 2, 16, 2>;  // BM = 64 rows, BN = 128 columns, 256 threads
constexpr int TM_ = 16, TN_ = 2, WN_ = 2;

template <int CWA, int CWB, bool CONV, int MODE>
int launch_gemm(const GemmArgs& g, cudaStream_t st) {
  auto kern = k_popc_gemm<Cfg, CWA, CWB, CONV, MODE, TM_, TN_, WN_>;
  static std::atomic<uint64_t> attr{0};
  smem_optin(kern, Cfg::SMEM, attr);
  if (g.M == 0 || g.N == 0) return 0;
  dim3 grid((unsigned)cdiv(g.M, Cfg::BM), (unsigned)cdiv(g.N, Cfg::BN));
  launch_k(kern, grid, 256, Cfg::SMEM, st, g);
  return launched();
}

template <bool CONV, int MODE>
int dispatch_cw(const GemmArgs& g, int cwa, int cwb, cudaStream_t st) {
#define B2_CASE(A, B) \
  if (cwa == A && cwb == B) return launch_gemm<A, B, CONV, MODE>(g, st);
  B2_CASE(4, 4) B2_CASE(4, 2) B2_CASE(2, 4) B2_CASE(2, 2) B2_CASE(1, 4) B2_CASE(1, 2)
#undef B2_CASE
  return B2_EINVAL;
}

// largest of {4, 2, 1} dividing both the word offset granularity and pitch
inline int chunk_words(int64_t a, int64_t b) {
  if (a % 4 == 0 && b % 4 == 0) return 4;
  if (a % 2 == 0 && b % 2 == 0) return 2;
  return 1;
}

// Batch-small dense (_kernels.py:109-117 bgemv_packed, batched over <= 8
// activation lines): a weight stream.  A block of 8 warps owns 32 units;
// each warp computes 4 of them with all their K-word loads in flight (lanes
// stride K for coalescing), reduces with __reduce_add_sync, and the block
// assembles the 32 results (PACK: one threshold word via ballot).
template <bool PACK>
__global__ void __launch_bounds__(256) k_dense_small(const uint32_t* __restrict__ x, int64_t batch, int64_t ldx,
                                                    const uint32_t* __restrict__ w, int64_t units, int64_t ldw,
                                                    int kw32, int32_t kbits, int32_t* __restrict__ out,
                                                    uint32_t* __restrict__ out_bits, int64_t ldo32,
                                                    const int32_t* __restrict__ thresh, const uint8_t* __restrict__ ge) {
  pdl_entry();
  __shared__ int32_t res[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ubase = (int64_t)blockIdx.x * 32;
  const int64_t u0 = ubase + warp * 4;
  for (int64_t bi = 0; bi < batch; ++bi) {
    const uint32_t* xr = x + bi * ldx;
    uint32_t part[4] = {0, 0, 0, 0};
#pragma unroll 4
    for (int k = lane; k < kw32; k += 32) {
      const uint32_t xv = __ldg(xr + k);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (u0 + i < units) part[i] += __popc(__ldg(w + (u0 + i) * ldw + k) ^ xv);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t tot = __reduce_add_sync(0xffffffffu, part[i]);
      if (lane == 0) res[warp * 4 + i] = kbits - 2 * (int32_t)tot;
    }
    __syncthreads();
    if (warp == 0) {
      const int64_t u = ubase + lane;
      const int32_t mine = res[lane];
      if constexpr (PACK) {
        const bool bit = u < units && thr_bit(mine, thresh[u < units ? u : 0], ge[u < units ? u : 0] != 0);
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        const int64_t widx = ubase >> 5;
        if (lane == 0 && widx < ldo32) out_bits[bi * ldo32 + widx] = word;
      } else {
        if (u < units) out[bi * units + u] = mine;
      }
    }
    __syncthreads();
  }
}

// _kernels.py:170-199 unroll_packed, batched.  One thread per output uint64
// word of an unrolled row; window cells are copied as bit runs.
__global__ void k_unroll(const uint64_t* __restrict__ lines, int64_t batch, int h, int w, int c, int kh, int kw,
                         int stride, int pad, int h_out, int w_out, int64_t row_words, uint64_t* __restrict__ out) {
  pdl_entry();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t rows = batch * h_out * w_out;
  if (t >= rows * row_words) return;
  int64_t row = t / row_words;
  int q = (int)(t - row * row_words);
  int64_t img = row / ((int64_t)h_out * w_out);
  int r = (int)(row - img * h_out * w_out);
  int i = r / w_out, j = r % w_out;
  const bool axis_channel = c > 1;
  const int64_t site_words = (c + 63) >> 6;
  const int64_t line_words = axis_channel ? site_words : (w + 63) >> 6;
  const int64_t img_words = axis_channel ? (int64_t)h * w * site_words : (int64_t)h * line_words;
  const uint64_t* src = lines + img * img_words;
  const int64_t k = (int64_t)kh * kw * c;
  int64_t lo = (int64_t)q * 64, hi = lo + 64 < k ? lo + 64 : k;
  uint64_t word = 0;
  for (int64_t cell = lo / c; cell * c < hi; ++cell) {
    int dy = (int)(cell / kw), dx = (int)(cell % kw);
    int ii = i * stride + dy - pad, jj = j * stride + dx - pad;
    if (ii < 0 || ii >= h || jj < 0 || jj >= w) continue;
    int64_t b0 = cell * c;  // first bit of the cell in the row
    int64_t s = b0 > lo ? b0 : lo, e = b0 + c < hi ? b0 + c : hi;
    uint64_t bits;
    if (axis_channel) {
      bits = get_bits64(src + ((int64_t)ii * w + jj) * site_words, s - b0, (int)(e - s));
    } else {
      bits = (src[(int64_t)ii * line_words + (jj >> 6)] >> (jj & 63)) & 1ULL;
    }
    word |= bits << (s - lo);
  }
  out[t] = word;
}

// layers.py:224-252 compute_correction: corr[pos, f] = sum of filter f's
// +/-1 weights over the window cells lying in the padding ring.
__global__ void k_correction(const uint64_t* __restrict__ wwords, int64_t filters, int h, int w, int c, int kh,
                             int kw, int stride, int pad, int h_out, int w_out, int32_t* __restrict__ corr) {
  pdl_entry();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)h_out * w_out * filters) return;
  int64_t pos = t / filters, f = t % filters;
  int i = (int)(pos / w_out), j = (int)(pos % w_out);
  const int64_t wpl = (((int64_t)kh * kw * c) + 63) >> 6;
  const uint64_t* line = wwords + f * wpl;
  int32_t s = 0;
  if (pad) {
    for (int dy = 0; dy < kh; ++dy)
      for (int dx = 0; dx < kw; ++dx) {
        int ii = i * stride + dy - pad, jj = j * stride + dx - pad;
        if (ii >= 0 && ii < h && jj >= 0 && jj < w) continue;
        int64_t b0 = (int64_t)(dy * kw + dx) * c;
        int ones = 0;
        for (int64_t o = 0; o < c; o += 64) {
          int len = c - o < 64 ? (int)(c - o) : 64;
          ones += __popcll(get_bits64(line, b0 + o, len));
        }
        s += 2 * ones - c;
      }
  }
  corr[t] = s;
}

inline void conv_geom(GemmArgs& g, const uint64_t* lines, int h, int w, int c, int kh, int kw, int stride, int pad) {
  g.a = (const uint32_t*)lines;
  g.lda = 0;
  g.H = h;
  g.W = w;
  g.spw = c / 32;
  g.sstride = (int)(2 * wpl64(c));
  g.kw_ = kw;
  g.stride = stride;
  g.pad = pad;
  g.Ho = (h + 2 * pad - kh) / stride + 1;
  g.Wo = (w + 2 * pad - kw) / stride + 1;
  g.kwords = kh * kw * g.spw;
  g.kbits = kh * kw * c;
}

}  // namespace b2

using namespace b2;

extern "C" {

int b2_bgemm(const uint64_t* a, int64_t m, const uint64_t* b, int64_t n, int64_t wpl, int32_t k, int32_t* out,
             void* stream) {
  if (m < 0 || n < 0 || wpl < 1 || k < 1 || k > 64 * wpl) return B2_EINVAL;
  GemmArgs g{};
  g.a = (const uint32_t*)a;
  g.lda = 2 * wpl;
  g.b = (const uint32_t*)b;
  g.ldb = 2 * wpl;
  g.kwords = (int)(2 * wpl);
  g.M = m;
  g.N = (int)n;
  g.kbits = k;
  g.out_i32 = out;
  g.ldo = n;
  int cw = chunk_words(2 * wpl, 2 * wpl);
  return dispatch_cw<false, EPI_I32>(g, cw, cw, S(stream));
}

int b2_bgemv(const uint64_t* w, int64_t units, int64_t wpl, const uint64_t* x, int64_t batch, int32_t k, int32_t* out,
             void* stream) {
  if (units < 0 || batch < 0 || wpl < 1 || k < 1 || k > 64 * wpl) return B2_EINVAL;
  if (!units || !batch) return 0;
  if (batch <= 8) {
    launch_k(k_dense_small<false>, (unsigned)cdiv(units, 32), 256, 0, S(stream), 
        (const uint32_t*)x, batch, 2 * wpl, (const uint32_t*)w, units, 2 * wpl, (int)(2 * wpl), k, out, nullptr, 0,
        nullptr, nullptr);
    return launched();
  }
  return b2_bgemm(x, batch, w, units, wpl, k, out, stream);
}

int b2_dense_bn_pack(const uint64_t* x, int64_t batch, const uint64_t* w, int64_t units, int64_t wpl, int32_t k,
                     b2_thresh th, uint64_t* out, void* stream) {
  if (units < 1 || batch < 0 || wpl < 1 || k < 1 || k > 64 * wpl || !th.thresh || !th.ge_dir) return B2_EINVAL;
  if (!batch) return 0;
  int64_t ldo32 = 2 * wpl64(units);
  if (batch <= 8) {
    // one block per output word, padding words included (they must be written as 0)
    launch_k(k_dense_small<true>, (unsigned)(cdiv(units, 32) > ldo32 ? cdiv(units, 32) : ldo32), 256, 0, S(stream), 
        (const uint32_t*)x, batch, 2 * wpl, (const uint32_t*)w, units, 2 * wpl, (int)(2 * wpl), k, nullptr,
        (uint32_t*)out, ldo32, th.thresh, th.ge_dir);
    return launched();
  }
  GemmArgs g{};
  g.a = (const uint32_t*)x;
  g.lda = 2 * wpl;
  g.b = (const uint32_t*)w;
  g.ldb = 2 * wpl;
  g.kwords = (int)(2 * wpl);
  g.M = batch;
  g.N = (int)units;
  g.kbits = k;
  g.out_bits = (uint32_t*)out;
  g.ldo32 = ldo32;
  g.thresh = th.thresh;
  g.ge = th.ge_dir;
  int cw = chunk_words(2 * wpl, 2 * wpl);
  return dispatch_cw<false, EPI_PACK>(g, cw, cw, S(stream));
}

int b2_unroll_packed(const uint64_t* lines, int64_t batch, int h, int w, int c, int kh, int kw, int stride, int pad,
                     uint64_t* out, void* stream) {
  if (batch < 0 || h < 1 || w < 1 || c < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0) return B2_EINVAL;
  if (h + 2 * pad < kh || w + 2 * pad < kw) return B2_EINVAL;
  int h_out = (h + 2 * pad - kh) / stride + 1, w_out = (w + 2 * pad - kw) / stride + 1;
  int64_t row_words = wpl64((int64_t)kh * kw * c);
  int64_t n = batch * h_out * w_out * row_words;
  if (!n) return 0;
  launch_k(k_unroll, (unsigned)cdiv(n, 256), 256, 0, S(stream), lines, batch, h, w, c, kh, kw, stride, pad, h_out, w_out,
                                                           row_words, out);
  return launched();
}

int b2_conv_correction(const uint64_t* wwords, int64_t filters, int h, int w, int c, int kh, int kw, int stride,
                       int pad, int32_t* corr, void* stream) {
  if (filters < 1 || h < 1 || w < 1 || c < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0) return B2_EINVAL;
  if (h + 2 * pad < kh || w + 2 * pad < kw) return B2_EINVAL;
  int h_out = (h + 2 * pad - kh) / stride + 1, w_out = (w + 2 * pad - kw) / stride + 1;
  int64_t n = (int64_t)h_out * w_out * filters;
  launch_k(k_correction, (unsigned)cdiv(n, 256), 256, 0, S(stream), wwords, filters, h, w, c, kh, kw, stride, pad, h_out,
                                                              w_out, corr);
  return launched();
}

int64_t b2_conv_scratch_words(int64_t batch, int h, int w, int c, int kh, int kw, int stride, int pad) {
  if (c % 32 == 0) return 0;
  int h_out = (h + 2 * pad - kh) / stride + 1, w_out = (w + 2 * pad - kw) / stride + 1;
  return batch * h_out * w_out * wpl64((int64_t)kh * kw * c);
}

int b2_conv_forward(const uint64_t* lines, int64_t batch, int h, int w, int c, const uint64_t* wwords,
                    int64_t filters, int kh, int kw, int stride, int pad, const int32_t* corr, uint64_t* scratch,
                    int32_t* out, void* stream) {
  if (batch < 0 || h < 1 || w < 1 || c < 1 || filters < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0)
    return B2_EINVAL;
  if (h + 2 * pad < kh || w + 2 * pad < kw) return B2_EINVAL;
  int64_t k = (int64_t)kh * kw * c, wpl = wpl64(k);
  GemmArgs g{};
  conv_geom(g, lines, h, w, c, kh, kw, stride, pad);
  g.b = (const uint32_t*)wwords;
  g.ldb = 2 * wpl;
  g.M = batch * g.Ho * g.Wo;
  g.N = (int)filters;
  g.corr = corr;
  g.out_i32 = out;
  g.ldo = filters;
  if (c % 32 == 0) {
    return dispatch_cw<true, EPI_I32>(g, chunk_words(g.spw, g.sstride), chunk_words(g.ldb, g.ldb), S(stream));
  }
  if (!scratch) return B2_EINVAL;
  int rc = b2_unroll_packed(lines, batch, h, w, c, kh, kw, stride, pad, scratch, stream);
  if (rc) return rc;
  // plain GEMM over the unrolled rows; correction indexed by row % (Ho*Wo)
  GemmArgs p{};
  p.a = (const uint32_t*)scratch;
  p.lda = 2 * wpl;
  p.b = (const uint32_t*)wwords;
  p.ldb = 2 * wpl;
  p.kwords = (int)(2 * wpl);
  p.M = g.M;
  p.N = (int)filters;
  p.kbits = (int32_t)k;
  p.out_i32 = out;
  p.ldo = filters;
  int cw = chunk_words(2 * wpl, 2 * wpl);
  rc = dispatch_cw<false, EPI_I32>(p, cw, cw, S(stream));
  if (rc || !corr) return rc;
  return b2_add_correction_i32(out, corr, g.M * filters, (int64_t)g.Ho * g.Wo * filters, stream);
}

int b2_conv_bn_pack(const uint64_t* lines, int64_t batch, int h, int w, int c, const uint64_t* wwords,
                    int64_t filters, int kh, int kw, int stride, int pad, const int32_t* corr, int pool, b2_thresh th,
                    uint64_t* out, void* stream) {
  if (batch < 0 || h < 1 || w < 1 || c < 1 || filters < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0)
    return B2_EINVAL;
  if (c % 32 || !th.thresh || !th.ge_dir) return B2_EINVAL;
  if (h + 2 * pad < kh || w + 2 * pad < kw) return B2_EINVAL;
  int64_t k = (int64_t)kh * kw * c, wpl = wpl64(k);
  GemmArgs g{};
  conv_geom(g, lines, h, w, c, kh, kw, stride, pad);
  if (pool && ((g.Ho & 1) || (g.Wo & 1))) return B2_EINVAL;
  g.b = (const uint32_t*)wwords;
  g.ldb = 2 * wpl;
  g.M = batch * g.Ho * g.Wo;
  g.N = (int)filters;
  g.corr = corr;
  g.out_bits = (uint32_t*)out;
  g.ldo32 = 2 * wpl64(filters);
  g.thresh = th.thresh;
  g.ge = th.ge_dir;
  int cwa = chunk_words(g.spw, g.sstride), cwb = chunk_words(g.ldb, g.ldb);
  if (pool) return dispatch_cw<true, EPI_POOLPACK>(g, cwa, cwb, S(stream));
  return dispatch_cw<true, EPI_PACK>(g, cwa, cwb, S(stream));
}

}  // extern "C"
