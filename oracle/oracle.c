/*
 * oracle.c — CPU restatement of the reference `bitnn` packed kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py; nothing in the product package
 * (paper_1705_07175_b200/) links, imports or calls it.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load liboracle.so.
 *
 * Each function restates one Numba kernel of the reference
 * (/root/reference/pkg/src/bitnn/_kernels.py) in plain C with the same
 * data layout: uint64 words, LSB-first, +1 -> bit 1, zero padding bits.
 * Parallel loops (`#pragma omp parallel for`) sit exactly where the
 * reference uses numba `prange`, so the CPU timing mirrors the
 * reference's own threading structure.  Floating-point code is compiled
 * with -ffp-contract=off (no FMA) like numpy/numba's separately rounded
 * operations.
 *
 * Parity is pinned by tests/test_oracle_golden.py against vectors that
 * tests/golden/make_golden.py produced by running the reference itself.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>

#define WPL(bits) (((bits) + 63) >> 6)

static inline int64_t popc64(uint64_t x) { return (int64_t)__builtin_popcountll(x); }

/* _kernels.py:43-54 pack_lines: bit = !(x < 0)  (0.0 and NaN -> 1) */
void o_pack_lines(const float* lines, int64_t n_lines, int64_t bits, uint64_t* out) {
  int64_t wpl = WPL(bits);
  memset(out, 0, sizeof(uint64_t) * n_lines * wpl);
#pragma omp parallel for schedule(static)
  for (int64_t li = 0; li < n_lines; ++li)
    for (int64_t b = 0; b < bits; ++b)
      if (!(lines[li * bits + b] < 0.0f)) out[li * wpl + (b >> 6)] |= 1ULL << (b & 63);
}

/* _kernels.py:57-64 unpack_lines */
void o_unpack_lines(const uint64_t* words, int64_t n_lines, int64_t bits, float* out) {
  int64_t wpl = WPL(bits);
#pragma omp parallel for schedule(static)
  for (int64_t li = 0; li < n_lines; ++li)
    for (int64_t b = 0; b < bits; ++b)
      out[li * bits + b] = ((words[li * wpl + (b >> 6)] >> (b & 63)) & 1ULL) ? 1.0f : -1.0f;
}

/* _kernels.py:67-82 pack_byte_planes: out (8, n_lines, wpl) */
void o_pack_byte_planes(const uint8_t* lines, int64_t n_lines, int64_t bits, uint64_t* out) {
  int64_t wpl = WPL(bits);
  memset(out, 0, sizeof(uint64_t) * 8 * n_lines * wpl);
#pragma omp parallel for schedule(static)
  for (int64_t li = 0; li < n_lines; ++li)
    for (int64_t b = 0; b < bits; ++b) {
      unsigned v = lines[li * bits + b];
      for (int p = 0; p < 8; ++p)
        if ((v >> p) & 1u) out[((int64_t)p * n_lines + li) * wpl + (b >> 6)] |= 1ULL << (b & 63);
    }
}

/* _kernels.py:85-106 bgemm_packed: out[m,n] = k - 2*popc(a_m ^ b_n); 64x64 tiles,
 * parallel over row tiles only (thread-count invariant). */
void o_bgemm(const uint64_t* a, int64_t m_total, const uint64_t* b, int64_t n_total, int64_t w_total,
             int32_t k, int32_t* out) {
  const int64_t TM = 64, TN = 64;
  int64_t n_row_tiles = (m_total + TM - 1) / TM;
#pragma omp parallel for schedule(static)
  for (int64_t mt = 0; mt < n_row_tiles; ++mt) {
    int64_t m0 = mt * TM, m1 = m0 + TM < m_total ? m0 + TM : m_total;
    for (int64_t n0 = 0; n0 < n_total; n0 += TN) {
      int64_t n1 = n0 + TN < n_total ? n0 + TN : n_total;
      for (int64_t m = m0; m < m1; ++m)
        for (int64_t n = n0; n < n1; ++n) {
          int64_t acc = 0;
          const uint64_t* ar = a + m * w_total;
          const uint64_t* br = b + n * w_total;
          for (int64_t w = 0; w < w_total; ++w) acc += popc64(ar[w] ^ br[w]);
          out[m * n_total + n] = k - 2 * (int32_t)acc;
        }
    }
  }
}

/* _kernels.py:109-117 bgemv_packed */
void o_bgemv(const uint64_t* a, int64_t m_total, int64_t w_total, const uint64_t* x, int32_t k, int32_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < m_total; ++m) {
    int64_t acc = 0;
    for (int64_t w = 0; w < w_total; ++w) acc += popc64(a[m * w_total + w] ^ x[w]);
    out[m] = k - 2 * (int32_t)acc;
  }
}

/* _kernels.py:120-127 count_plane_bits */
void o_count_plane_bits(const uint64_t* planes, int64_t wpl, int64_t* out) {
  for (int p = 0; p < 8; ++p) {
    int64_t acc = 0;
    for (int64_t w = 0; w < wpl; ++w) acc += popc64(planes[p * wpl + w]);
    out[p] = acc;
  }
}

/* _kernels.py:130-147 bitplane_matvec: sum_p 2^p (2 popc(plane_p & w) - popc(plane_p)) */
void o_bitplane_matvec(const uint64_t* planes, const int64_t* pops, const uint64_t* w, int64_t units,
                       int64_t w_total, int64_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < units; ++u) {
    int64_t acc = 0;
    for (int p = 0; p < 8; ++p) {
      int64_t m = 0;
      for (int64_t x = 0; x < w_total; ++x) m += popc64(planes[p * w_total + x] & w[u * w_total + x]);
      acc += (2 * m - pops[p]) * ((int64_t)1 << p);
    }
    out[u] = acc;
  }
}

/* _kernels.py:150-167 _or_bits */
static inline void or_bits(const uint64_t* src, int64_t n_src_words, uint64_t* dst_row, int64_t row_words,
                           int64_t dst_bit0) {
  int64_t dw = dst_bit0 >> 6;
  unsigned db = (unsigned)(dst_bit0 & 63);
  if (db == 0) {
    for (int64_t w = 0; w < n_src_words; ++w) dst_row[dw + w] |= src[w];
  } else {
    unsigned inv = 64 - db;
    for (int64_t w = 0; w < n_src_words; ++w) {
      uint64_t v = src[w];
      dst_row[dw + w] |= v << db;
      if (dw + w + 1 < row_words) dst_row[dw + w + 1] |= v >> inv;
    }
  }
}

/* _kernels.py:170-199 unroll_packed (bit im2col; OOB sites stay 0 bits) */
void o_unroll_packed(const uint64_t* lines, int h, int w, int c, int axis_channel, int kh, int kw, int stride,
                     int pad, uint64_t* out) {
  int h_out = (h + 2 * pad - kh) / stride + 1;
  int w_out = (w + 2 * pad - kw) / stride + 1;
  int64_t site_words = (c + 63) >> 6;
  int64_t k = (int64_t)kh * kw * c;
  int64_t row_words = WPL(k);
  int64_t line_words = axis_channel ? site_words : WPL(w);
  memset(out, 0, sizeof(uint64_t) * (int64_t)h_out * w_out * row_words);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)h_out * w_out; ++r) {
    int i = (int)(r / w_out), j = (int)(r % w_out);
    uint64_t* row = out + r * row_words;
    for (int dy = 0; dy < kh; ++dy) {
      int ii = i * stride + dy - pad;
      if (ii < 0 || ii >= h) continue;
      for (int dx = 0; dx < kw; ++dx) {
        int jj = j * stride + dx - pad;
        if (jj < 0 || jj >= w) continue;
        int64_t bit0 = (int64_t)(dy * kw + dx) * c;
        if (axis_channel) {
          or_bits(lines + ((int64_t)ii * w + jj) * line_words, site_words, row, row_words, bit0);
        } else {
          uint64_t bit = (lines[(int64_t)ii * line_words + (jj >> 6)] >> (jj & 63)) & 1ULL;
          if (bit) row[bit0 >> 6] |= 1ULL << (bit0 & 63);
        }
      }
    }
  }
}

/* _kernels.py:224-240 maxpool (int32 HWC, floor arithmetic) */
void o_maxpool_i32(const int32_t* x, int h, int w, int c, int ph, int pw, int stride, int32_t* out) {
  int h_out = (h - ph) / stride + 1, w_out = (w - pw) / stride + 1;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)h_out * w_out; ++r) {
    int i = (int)(r / w_out), j = (int)(r % w_out);
    for (int ch = 0; ch < c; ++ch) {
      int32_t best = x[((int64_t)(i * stride) * w + j * stride) * c + ch];
      for (int dy = 0; dy < ph; ++dy)
        for (int dx = 0; dx < pw; ++dx) {
          int32_t v = x[((int64_t)(i * stride + dy) * w + (j * stride + dx)) * c + ch];
          if (v > best) best = v;
        }
      out[((int64_t)i * w_out + j) * c + ch] = best;
    }
  }
}

/* _kernels.py:243-267 threshold_sign_pack (serial in the reference).
 * x is read through `xkind`: 0 = int32, 1 = int64, 2 = uint8. */
static inline int64_t load_x(const void* x, int xkind, int64_t i) {
  if (xkind == 0) return ((const int32_t*)x)[i];
  if (xkind == 1) return ((const int64_t*)x)[i];
  return ((const uint8_t*)x)[i];
}

void o_threshold_sign_pack(const void* x, int xkind, int64_t sites, int64_t c, const int64_t* thresh,
                           const uint8_t* ge_dir, int flat, uint64_t* out) {
  int64_t out_words = flat ? WPL(sites * c) : sites * WPL(c);
  int64_t wpl = WPL(c);
  memset(out, 0, sizeof(uint64_t) * out_words);
  for (int64_t s = 0; s < sites; ++s)
    for (int64_t ch = 0; ch < c; ++ch) {
      int64_t v = load_x(x, xkind, s * c + ch);
      int64_t t = thresh[ch];
      int bit = ge_dir[ch] ? (v >= t) : (v <= t);
      if (bit) {
        if (flat) {
          int64_t k = s * c + ch;
          out[k >> 6] |= 1ULL << (k & 63);
        } else {
          out[s * wpl + (ch >> 6)] |= 1ULL << (ch & 63);
        }
      }
    }
}

/* _kernels.py:285-295 bn_affine: (float64(x) - mean) * scale + beta, no FMA */
void o_bn_affine(const void* x, int xkind, int64_t n, const double* mean, const double* scale, const double* beta,
                 int64_t c, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t ch = i % c;
    volatile double d = (double)load_x(x, xkind, i) - mean[ch];
    volatile double e = d * scale[ch];
    out[i] = e + beta[ch];
  }
}

/* layers.py:137-140, 143-191 BatchNormLayer float64 working form + _calibrate.
 * Writes scale64 and the int64 threshold / ge_dir per channel. */
#define ALWAYS (-(1LL << 62))
#define NEVER (1LL << 62)
#define SEARCH_BOUND (1LL << 40)

static inline double bn_eval(double x, double mean, double scale, double beta) {
  volatile double d = x - mean;
  volatile double e = d * scale;
  return e + beta;
}

void o_bn_calibrate(const float* mean, const float* var, const float* gamma, const float* beta, double eps,
                    int64_t channels, double* scale64, int64_t* thresh, uint8_t* ge_dir) {
  for (int64_t c = 0; c < channels; ++c) {
    double m = (double)mean[c], b = (double)beta[c];
    volatile double den = sqrt((double)var[c] + eps);
    double s = (double)gamma[c] / den;
    scale64[c] = s;
    if (s == 0.0) {
      thresh[c] = b >= 0 ? ALWAYS : NEVER;
      ge_dir[c] = 1;
      continue;
    }
    int64_t lo = -SEARCH_BOUND, hi = SEARCH_BOUND;
    if (s > 0) {
      ge_dir[c] = 1;
      if (bn_eval((double)lo, m, s, b) >= 0) thresh[c] = ALWAYS;
      else if (bn_eval((double)hi, m, s, b) < 0) thresh[c] = NEVER;
      else {
        while (hi - lo > 1) {
          int64_t mid = lo + ((hi - lo) >> 1);
          /* python (lo + hi) // 2 is floor division; lo + (hi-lo)/2 is identical for hi > lo */
          if (bn_eval((double)mid, m, s, b) >= 0) hi = mid; else lo = mid;
        }
        thresh[c] = hi;
      }
    } else {
      ge_dir[c] = 0;
      if (bn_eval((double)hi, m, s, b) >= 0) thresh[c] = NEVER;
      else if (bn_eval((double)lo, m, s, b) < 0) thresh[c] = ALWAYS;
      else {
        while (hi - lo > 1) {
          int64_t mid = lo + ((hi - lo) >> 1);
          if (bn_eval((double)mid, m, s, b) >= 0) lo = mid; else hi = mid;
        }
        thresh[c] = lo;
      }
    }
  }
}

/* layers.py:224-252 compute_correction from packed filter lines (F, wpl(kh*kw*c)) */
void o_compute_correction(const uint64_t* wwords, int64_t filters, int h, int w, int c, int kh, int kw,
                          int stride, int pad, int32_t* corr) {
  int h_out = (h + 2 * pad - kh) / stride + 1;
  int w_out = (w + 2 * pad - kw) / stride + 1;
  int64_t k = (int64_t)kh * kw * c, wpl = WPL(k);
  memset(corr, 0, sizeof(int32_t) * (int64_t)h_out * w_out * filters);
  if (pad == 0) return;
  for (int i = 0; i < h_out; ++i)
    for (int j = 0; j < w_out; ++j)
      for (int dy = 0; dy < kh; ++dy) {
        int ii = i * stride + dy - pad;
        for (int dx = 0; dx < kw; ++dx) {
          int jj = j * stride + dx - pad;
          if (ii < 0 || ii >= h || jj < 0 || jj >= w) {
            int64_t base = (int64_t)(dy * kw + dx) * c;
            for (int64_t f = 0; f < filters; ++f) {
              int32_t s = 0;
              for (int64_t ch = 0; ch < c; ++ch) {
                int64_t bb = base + ch;
                s += ((wwords[f * wpl + (bb >> 6)] >> (bb & 63)) & 1ULL) ? 1 : -1;
              }
              corr[((int64_t)i * w_out + j) * filters + f] += s;
            }
          }
        }
      }
}

/* network.py:193-198 _PackedConv.run: acc (+)= correction, elementwise */
void o_add_i32(int32_t* acc, const int32_t* corr, int64_t n) {
  for (int64_t i = 0; i < n; ++i) acc[i] += corr[i];
}

int o_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
