// Stand-alone epilogue kernels: max-pool, batchnorm-threshold + sign + pack,
// final float64 batchnorm, on-device batchnorm calibration, correction add
// (SURVEY.md §8 a-9, a-11 .. a-14).  The fused GEMM epilogues in
// gemm_popc.cuh cover the common network shapes; these kernels implement
// the general layouts (flat packing with C % 64 != 0, column-axis lines,
// int64 / uint8 inputs, non-2x2 pooling) bit-exactly.
#include "common.cuh"

namespace b2 {

// _kernels.py:224-240 maxpool, batched int32 (batch, h, w, c)
__global__ void k_maxpool_i32(const int32_t* __restrict__ x, int64_t batch, int h, int w, int c, int ph, int pw,
                              int stride, int h_out, int w_out, int32_t* __restrict__ out) {
  pdl_entry();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = batch * h_out * w_out * c;
  if (t >= total) return;
  int ch = (int)(t % c);
  int64_t r = t / c;
  int j = (int)(r % w_out);
  r /= w_out;
  int i = (int)(r % h_out);
  int64_t img = r / h_out;
  const int32_t* xi = x + img * h * w * c;
  int32_t best = xi[((int64_t)(i * stride) * w + j * stride) * c + ch];
  for (int dy = 0; dy < ph; ++dy)
    for (int dx = 0; dx < pw; ++dx) {
      int32_t v = xi[((int64_t)(i * stride + dy) * w + (j * stride + dx)) * c + ch];
      best = v > best ? v : best;
    }
  out[t] = best;
}

template <typename T>
__device__ __forceinline__ int64_t ld_as_i64(const void* x, int64_t i) {
  return (int64_t)static_cast<const T*>(x)[i];
}
template <typename T>
__device__ __forceinline__ double ld_as_f64(const void* x, int64_t i) {
  return (double)static_cast<const T*>(x)[i];
}

// _kernels.py:243-267 threshold_sign_pack, batched.  One warp per output
// 32-bit word: lane i decides bit i, ballot assembles the word.
template <typename T>
__global__ void k_threshold_pack(const void* __restrict__ x, int64_t batch, int64_t sites, int64_t c,
                                 const int64_t* __restrict__ thresh, const uint8_t* __restrict__ ge, int flat,
                                 int64_t line_words32, int64_t lines_per_img, uint32_t* __restrict__ out) {
  pdl_entry();
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t words = batch * lines_per_img * line_words32;
  if (warp >= words) return;
  int lane = threadIdx.x & 31;
  int64_t img = warp / (lines_per_img * line_words32);
  int64_t rem = warp - img * lines_per_img * line_words32;
  int64_t line = rem / line_words32, q = rem % line_words32;
  int64_t b = q * 32 + lane;  // bit within the line
  bool bit = false;
  int64_t s, ch;
  if (flat) {
    s = b / c;
    ch = b - s * c;
    bit = s < sites;
  } else {
    s = line;
    ch = b;
    bit = ch < c;
  }
  if (bit) {
    int64_t v = ld_as_i64<T>(x, (img * sites + s) * c + ch);
    int64_t t = thresh[ch];
    bit = ge[ch] ? (v >= t) : (v <= t);
  }
  uint32_t word = __ballot_sync(0xffffffffu, bit);
  if (lane == 0) out[warp] = word;
}

// _kernels.py:285-295 bn_affine: three separately rounded float64 ops
template <typename T>
__global__ void k_bn_affine(const void* __restrict__ x, int64_t n, const double* __restrict__ mean,
                            const double* __restrict__ scale, const double* __restrict__ beta, int64_t c,
                            double* __restrict__ out) {
  pdl_entry();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t ch = i % c;
  double d = __dsub_rn(ld_as_f64<T>(x, i), mean[ch]);
  out[i] = __dadd_rn(__dmul_rn(d, scale[ch]), beta[ch]);
}

__device__ __forceinline__ double bn_eval(double x, double m, double s, double b) {
  return __dadd_rn(__dmul_rn(__dsub_rn(x, m), s), b);
}

// layers.py:137-191: scale64 = gamma / sqrt(var + eps) in float64 and the
// integer threshold by the same binary search, one thread per channel.
__global__ void k_bn_calibrate(const float* __restrict__ mean, const float* __restrict__ var,
                               const float* __restrict__ gamma, const float* __restrict__ beta, double eps, int64_t c,
                               int64_t bound, double* __restrict__ scale64, int64_t* __restrict__ thresh64,
                               uint8_t* __restrict__ ge_dir, int32_t* __restrict__ thresh32) {
  pdl_entry();
  int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= c) return;
  const int64_t ALWAYS = -(1LL << 62), NEVER = 1LL << 62, SB = 1LL << 40;
  double m = (double)mean[ch], b = (double)beta[ch];
  double s = __ddiv_rn((double)gamma[ch], __dsqrt_rn(__dadd_rn((double)var[ch], eps)));
  if (scale64) scale64[ch] = s;
  int64_t t;
  uint8_t ge;
  int64_t lo = -SB, hi = SB;
  if (s == 0.0) {
    t = b >= 0 ? ALWAYS : NEVER;
    ge = 1;
  } else if (s > 0) {
    ge = 1;
    if (bn_eval((double)lo, m, s, b) >= 0) t = ALWAYS;
    else if (bn_eval((double)hi, m, s, b) < 0) t = NEVER;
    else {
      while (hi - lo > 1) {
        int64_t mid = lo + ((hi - lo) >> 1);  // == floor((lo + hi) / 2)
        if (bn_eval((double)mid, m, s, b) >= 0) hi = mid; else lo = mid;
      }
      t = hi;
    }
  } else {
    ge = 0;
    if (bn_eval((double)hi, m, s, b) >= 0) t = NEVER;
    else if (bn_eval((double)lo, m, s, b) < 0) t = ALWAYS;
    else {
      while (hi - lo > 1) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (bn_eval((double)mid, m, s, b) >= 0) lo = mid; else hi = mid;
      }
      t = lo;
    }
  }
  thresh64[ch] = t;
  ge_dir[ch] = ge;
  if (thresh32) {
    int64_t cl = t < -(bound + 1) ? -(bound + 1) : (t > bound + 1 ? bound + 1 : t);
    thresh32[ch] = (int32_t)cl;
  }
}

__global__ void k_add_corr(int32_t* __restrict__ acc, const int32_t* __restrict__ corr, int64_t n, int64_t per) {
  pdl_entry();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) acc[i] += corr[i % per];
}

}  // namespace b2

using namespace b2;

extern "C" {

int b2_maxpool_i32(const int32_t* x, int64_t batch, int h, int w, int c, int ph, int pw, int stride, int32_t* out,
                   void* stream) {
  if (batch < 0 || h < ph || w < pw || ph < 1 || pw < 1 || stride < 1 || c < 1) return B2_EINVAL;
  int h_out = (h - ph) / stride + 1, w_out = (w - pw) / stride + 1;
  int64_t n = batch * h_out * w_out * c;
  if (!n) return 0;
  launch_k(k_maxpool_i32, (unsigned)cdiv(n, 256), 256, 0, S(stream), x, batch, h, w, c, ph, pw, stride, h_out, w_out, out);
  return launched();
}

int b2_threshold_pack(const void* x, int xkind, int64_t batch, int64_t sites, int64_t c, b2_thresh th, int flat,
                      uint64_t* out, void* stream) {
  if (batch < 0 || sites < 1 || c < 1 || !th.thresh64 || !th.ge_dir || xkind < 0 || xkind > 2) return B2_EINVAL;
  int64_t lines = flat ? 1 : sites;
  int64_t lw32 = 2 * wpl64(flat ? sites * c : c);
  int64_t words = batch * lines * lw32;
  if (!words) return 0;
  unsigned grid = (unsigned)cdiv(words, 8);
  cudaStream_t st = S(stream);
  if (xkind == 0)
    launch_k(k_threshold_pack<int32_t>, grid, 256, 0, st, x, batch, sites, c, th.thresh64, th.ge_dir, flat, lw32, lines,
                                                    (uint32_t*)out);
  else if (xkind == 1)
    launch_k(k_threshold_pack<int64_t>, grid, 256, 0, st, x, batch, sites, c, th.thresh64, th.ge_dir, flat, lw32, lines,
                                                    (uint32_t*)out);
  else
    launch_k(k_threshold_pack<uint8_t>, grid, 256, 0, st, x, batch, sites, c, th.thresh64, th.ge_dir, flat, lw32, lines,
                                                    (uint32_t*)out);
  return launched();
}

int b2_bn_affine_f64(const void* x, int xkind, int64_t n, const double* mean, const double* scale,
                     const double* beta, int64_t c, double* out, void* stream) {
  if (n < 0 || c < 1 || xkind < 0 || xkind > 3 || xkind == 2) return B2_EINVAL;
  if (!n) return 0;
  unsigned grid = (unsigned)cdiv(n, 256);
  if (xkind == 0)
    launch_k(k_bn_affine<int32_t>, grid, 256, 0, S(stream), x, n, mean, scale, beta, c, out);
  else if (xkind == 1)
    launch_k(k_bn_affine<int64_t>, grid, 256, 0, S(stream), x, n, mean, scale, beta, c, out);
  else
    launch_k(k_bn_affine<double>, grid, 256, 0, S(stream), x, n, mean, scale, beta, c, out);
  return launched();
}

int b2_bn_calibrate(const float* mean, const float* var, const float* gamma, const float* beta, double eps, int64_t c,
                    int64_t bound, double* scale64, int64_t* thresh64, uint8_t* ge_dir, int32_t* thresh32,
                    void* stream) {
  if (c < 1 || bound < 0 || bound > (1LL << 31) - 2 || !thresh64 || !ge_dir) return B2_EINVAL;
  launch_k(k_bn_calibrate, (unsigned)cdiv(c, 128), 128, 0, S(stream), mean, var, gamma, beta, eps, c, bound, scale64,
                                                                thresh64, ge_dir, thresh32);
  return launched();
}

int b2_add_correction_i32(int32_t* acc, const int32_t* corr, int64_t n, int64_t per_image, void* stream) {
  if (n < 0 || per_image < 1) return B2_EINVAL;
  if (!n) return 0;
  launch_k(k_add_corr, (unsigned)cdiv(n, 256), 256, 0, S(stream), acc, corr, n, per_image);
  return launched();
}

}  // extern "C"
