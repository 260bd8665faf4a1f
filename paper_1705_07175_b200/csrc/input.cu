// First-layer kernels: byte inputs (SURVEY.md §8 a-4, a-5, a-13 byte BN).
//
//  * k_input8_bn_pack: BMLP input layer.  Bit-plane decomposition of the
//    uint8 images happens in shared memory (8 ballots per 32 bytes), then an
//    AND-popc GEMM against the +/-1 weight rows:
//        y = sum_p 2^p (2 popc(plane_p & w) - popc(plane_p))
//          = 2 * sum_p 2^p popc(plane_p & w) - sum(bytes)     (gemm.py:120-146)
//    followed by the batchnorm threshold and a ballot repack.
//  * k_byte_conv_bn_pack: BCNN input layer.  Byte batchnorm thresholds
//    (network.py:128-138) build 3-bit sites in shared memory; each output
//    position's window (<= 32 bits) is XOR-popc'ed against every filter with
//    the out-of-bounds cells masked (== pad-as--1 + correction map), then
//    batchnorm threshold + ballot repack.
#include "common.cuh"

namespace b2 {

constexpr int I8_IMG = 32;   // images per CTA
constexpr int I8_TM = 4;     // images per warp
constexpr int I8_TN = 4;     // 32-unit groups per lane -> 128 units per CTA
constexpr int I8_MAXKW = 128;  // uint32 words of K held in shared memory (K <= 4096)

__global__ void __launch_bounds__(256) k_input8_bn_pack(const uint8_t* __restrict__ x, int64_t batch, int k,
                                                       int kw32, const uint32_t* __restrict__ w, int64_t units,
                                                       int64_t ldw, const int32_t* __restrict__ thresh,
                                                       const uint8_t* __restrict__ ge, uint32_t* __restrict__ out,
                                                       int64_t ldo32) {
  pdl_entry();
  extern __shared__ uint32_t sm[];
  const int pitchw = kw32 | 1;  // odd pitch: lanes hit distinct banks
  uint32_t* P = sm;                                   // [I8_IMG][8][kw32]
  uint32_t* Wt = P + I8_IMG * 8 * kw32;               // [128][pitchw]
  int32_t* Ssum = (int32_t*)(Wt + 32 * I8_TN * pitchw);  // [I8_IMG]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t img0 = (int64_t)blockIdx.x * I8_IMG;
  const int64_t u0 = (int64_t)blockIdx.y * 32 * I8_TN;

  // bit planes + byte sums of this CTA's images
  for (int ii = warp; ii < I8_IMG; ii += 8) {
    int64_t img = img0 + ii;
    int32_t bsum = 0;
    for (int q = 0; q < kw32; ++q) {
      int b = q * 32 + lane;
      unsigned v = (img < batch && b < k) ? x[img * k + b] : 0u;
      bsum += (int32_t)v;
      uint32_t mine = 0;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        uint32_t word = __ballot_sync(0xffffffffu, (v >> p) & 1u);
        if (lane == p) mine = word;
      }
      if (lane < 8) P[(ii * 8 + lane) * kw32 + q] = mine;
    }
    bsum = __reduce_add_sync(0xffffffffu, bsum);
    if (lane == 0) Ssum[ii] = bsum;
  }
  // weight rows of this CTA's 128 units
  for (int idx = threadIdx.x; idx < 32 * I8_TN * kw32; idx += 256) {
    int r = idx / kw32, q = idx - r * kw32;
    int64_t u = u0 + r;
    Wt[r * pitchw + q] = u < units ? w[u * ldw + q] : 0u;
  }
  __syncthreads();

  uint32_t acc[I8_TM][I8_TN];
#pragma unroll
  for (int i = 0; i < I8_TM; ++i)
#pragma unroll
    for (int j = 0; j < I8_TN; ++j) acc[i][j] = 0;
  const uint32_t* pw = P + (warp * I8_TM) * 8 * kw32;
  for (int q = 0; q < kw32; ++q) {
    uint32_t bw[I8_TN];
#pragma unroll
    for (int j = 0; j < I8_TN; ++j) bw[j] = Wt[(32 * j + lane) * pitchw + q];
#pragma unroll
    for (int i = 0; i < I8_TM; ++i)
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        uint32_t pv = pw[(i * 8 + p) * kw32 + q];
#pragma unroll
        for (int j = 0; j < I8_TN; ++j) acc[i][j] += (uint32_t)__popc(pv & bw[j]) << p;
      }
  }

#pragma unroll
  for (int i = 0; i < I8_TM; ++i) {
    int ii = warp * I8_TM + i;
    int64_t img = img0 + ii;
    int32_t s = Ssum[ii];
#pragma unroll
    for (int j = 0; j < I8_TN; ++j) {
      int64_t u = u0 + 32 * j + lane;
      bool bit = false;
      if (u < units) bit = thr_bit(2 * (int32_t)acc[i][j] - s, thresh[u], ge[u] != 0);
      uint32_t word = __ballot_sync(0xffffffffu, bit);
      int64_t widx = (u0 >> 5) + j;
      if (img < batch && widx < ldo32 && lane == ((i * I8_TN + j) & 31)) out[img * ldo32 + widx] = word;
    }
  }
}

// Generic batched bit-plane matvec (int64 out): one thread per (image, unit).
// planes are laid out (8, batch, wpl) as produced by b2_pack_byte_planes.
__global__ void k_bitplane_gemv(const uint64_t* __restrict__ planes, int64_t batch, const uint64_t* __restrict__ w,
                                int64_t units, int64_t wpl, int64_t* __restrict__ out) {
  pdl_entry();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch * units) return;
  int64_t img = t / units, u = t % units;
  const uint64_t* wr = w + u * wpl;
  int64_t acc = 0;
  for (int p = 0; p < 8; ++p) {
    const uint64_t* pl = planes + ((int64_t)p * batch + img) * wpl;
    int64_t m = 0, pop = 0;
    for (int64_t q = 0; q < wpl; ++q) {
      uint64_t v = pl[q];
      m += __popcll(v & wr[q]);
      pop += __popcll(v);
    }
    acc += (2 * m - pop) << p;
  }
  out[t] = acc;
}

__global__ void __launch_bounds__(256) k_byte_conv_bn_pack(const uint8_t* __restrict__ x, int h, int w, int c,
                                                          const int32_t* __restrict__ tin, const uint8_t* __restrict__ gin,
                                                          const uint32_t* __restrict__ wwords, int64_t ldw,
                                                          int filters, int kh, int kw, int stride, int pad, int h_out,
                                                          int w_out, const int32_t* __restrict__ tout,
                                                          const uint8_t* __restrict__ gout, uint32_t* __restrict__ out,
                                                          int ldo32) {
  pdl_entry();
  extern __shared__ uint32_t sm[];
  uint32_t* sites = sm;                 // [h*w] c-bit site codes
  uint32_t* wf = sites + h * w;         // [ngroups*32] filter words
  int32_t* tf = (int32_t*)(wf + ldo32 * 32);
  uint8_t* gf = (uint8_t*)(tf + ldo32 * 32);
  const int64_t img = blockIdx.x;
  const uint8_t* xi = x + img * (int64_t)h * w * c;
  for (int s = threadIdx.x; s < h * w; s += blockDim.x) {
    uint32_t code = 0;
    for (int ch = 0; ch < c; ++ch) {
      int32_t v = xi[s * c + ch];
      code |= (uint32_t)thr_bit(v, tin[ch], gin[ch] != 0) << ch;
    }
    sites[s] = code;
  }
  for (int f = threadIdx.x; f < ldo32 * 32; f += blockDim.x) {
    bool ok = f < filters;
    wf[f] = ok ? wwords[f * ldw] : 0u;
    tf[f] = ok ? tout[f] : 0;
    gf[f] = ok ? gout[f] : 1;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cmask = (c >= 32) ? 0xffffffffu : ((1u << c) - 1u);
  const int ngroups = (filters + 31) >> 5;
  for (int pos = warp; pos < h_out * w_out; pos += blockDim.x >> 5) {
    int i = pos / w_out, j = pos - (pos / w_out) * w_out;
    uint32_t win = 0, inmask = 0;
    for (int dy = 0; dy < kh; ++dy) {
      int ii = i * stride + dy - pad;
      for (int dx = 0; dx < kw; ++dx) {
        int jj = j * stride + dx - pad;
        if (ii < 0 || ii >= h || jj < 0 || jj >= w) continue;
        int sh = (dy * kw + dx) * c;
        win |= sites[ii * w + jj] << sh;
        inmask |= cmask << sh;
      }
    }
    const int nin = __popc(inmask);
    uint32_t mine = 0;
    for (int g = 0; g < ngroups; ++g) {
      int f = 32 * g + lane;
      int32_t dot = nin - 2 * __popc((win ^ wf[f]) & inmask);
      bool bit = f < filters && thr_bit(dot, tf[f], gf[f] != 0);
      uint32_t word = __ballot_sync(0xffffffffu, bit);
      if (lane == g) mine = word;
    }
    if (lane < ldo32) out[(img * h_out * w_out + pos) * ldo32 + lane] = mine;
  }
}

}  // namespace b2

using namespace b2;

extern "C" {

int b2_input8_bn_pack(const uint8_t* x, int64_t batch, int64_t k, const uint64_t* w, int64_t units, b2_thresh th,
                      uint64_t* out, void* stream) {
  if (batch < 0 || k < 1 || units < 1 || !th.thresh || !th.ge_dir) return B2_EINVAL;
  int kw32 = (int)(2 * wpl64(k));
  if (kw32 > I8_MAXKW) return B2_EINVAL;
  if (!batch) return 0;
  int pitchw = kw32 | 1;
  size_t smem = sizeof(uint32_t) * ((size_t)I8_IMG * 8 * kw32 + 32 * I8_TN * pitchw + I8_IMG);
  static std::atomic<uint64_t> attr{0};
  smem_optin(k_input8_bn_pack, 200 * 1024, attr);
  dim3 grid((unsigned)cdiv(batch, I8_IMG), (unsigned)cdiv(units, 32 * I8_TN));
  launch_k(k_input8_bn_pack, grid, 256, smem, S(stream), x, batch, (int)k, kw32, (const uint32_t*)w, units, kw32,
                                                   th.thresh, th.ge_dir, (uint32_t*)out, 2 * wpl64(units));
  return launched();
}

int b2_bitplane_gemv(const uint64_t* planes, int64_t batch, const uint64_t* w, int64_t units, int64_t wpl,
                     int64_t* out, void* stream) {
  if (batch < 0 || units < 0 || wpl < 1) return B2_EINVAL;
  int64_t n = batch * units;
  if (!n) return 0;
  launch_k(k_bitplane_gemv, (unsigned)cdiv(n, 256), 256, 0, S(stream), planes, batch, w, units, wpl, out);
  return launched();
}

int b2_byte_conv_bn_pack(const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in,
                         const uint64_t* wwords, int64_t filters, int kh, int kw, int stride, int pad,
                         b2_thresh th_out, uint64_t* out, void* stream) {
  if (batch < 0 || h < 1 || w < 1 || c < 1 || filters < 1 || filters > 1024 || kh < 1 || kw < 1 || stride < 1 ||
      pad < 0)
    return B2_EINVAL;
  if ((int64_t)kh * kw * c > 32 || !th_in.thresh || !th_in.ge_dir || !th_out.thresh || !th_out.ge_dir)
    return B2_EINVAL;
  if (h + 2 * pad < kh || w + 2 * pad < kw) return B2_EINVAL;
  if (!batch) return 0;
  int h_out = (h + 2 * pad - kh) / stride + 1, w_out = (w + 2 * pad - kw) / stride + 1;
  int ldo32 = (int)(2 * wpl64(filters));
  size_t smem = sizeof(uint32_t) * ((size_t)h * w + 2 * ldo32 * 32) + ldo32 * 32;
  if (smem > 200 * 1024) return B2_EINVAL;
  static std::atomic<uint64_t> attr{0};
  smem_optin(k_byte_conv_bn_pack, 200 * 1024, attr);
  int64_t ldw = 2 * wpl64((int64_t)kh * kw * c);
  launch_k(k_byte_conv_bn_pack, (unsigned)batch, 256, smem, S(stream), x, h, w, c, th_in.thresh, th_in.ge_dir,
                                                                 (const uint32_t*)wwords, ldw, (int)filters, kh, kw,
                                                                 stride, pad, h_out, w_out, th_out.thresh,
                                                                 th_out.ge_dir, (uint32_t*)out, ldo32);
  return launched();
}

}  // extern "C"
