// Sign-binarize / bit-pack kernels.
//
// One warp builds one 32-bit word with __ballot_sync: lane i owns element
// 32*j + i, so ballot bit i is element i of the word — exactly the
// reference's LSB-first order (_kernels.py:6-9).  Lines are padded to whole
// uint64 words; lanes past the line length vote 0, so padding bits are zero.
#include "common.cuh"

namespace b2 {

std::atomic<int64_t> g_launches{0};

// _kernels.py:43-54 pack_lines: bit = !(x < 0)  (0.0, -0.0 and NaN -> 1)
__global__ void k_pack_lines_f32(const float* __restrict__ lines, int64_t n_lines, int64_t bits, int64_t wpl32,
                                 uint32_t* __restrict__ out) {
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t total = n_lines * wpl32;
  if (warp >= total) return;
  int64_t line = warp / wpl32, j = warp % wpl32;
  int64_t b = j * 32 + lane_id();
  bool bit = false;
  if (b < bits) bit = !(lines[line * bits + b] < 0.0f);
  uint32_t w = __ballot_sync(0xffffffffu, bit);
  if (lane_id() == 0) out[warp] = w;
}

// _kernels.py:57-64 unpack_lines
__global__ void k_unpack_lines_f32(const uint32_t* __restrict__ words, int64_t n_lines, int64_t bits, int64_t wpl32,
                                   float* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lines * bits) return;
  int64_t line = i / bits, b = i % bits;
  out[i] = ((words[line * wpl32 + (b >> 5)] >> (b & 31)) & 1u) ? 1.0f : -1.0f;
}

// _kernels.py:67-82 pack_byte_planes: one warp -> 8 plane words
__global__ void k_pack_byte_planes(const uint8_t* __restrict__ lines, int64_t n_lines, int64_t bits, int64_t wpl32,
                                   uint32_t* __restrict__ out) {
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (warp >= n_lines * wpl32) return;
  int64_t line = warp / wpl32, j = warp % wpl32;
  int64_t b = j * 32 + lane_id();
  unsigned v = b < bits ? lines[line * bits + b] : 0u;
  uint32_t mine = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    uint32_t w = __ballot_sync(0xffffffffu, (v >> p) & 1u);
    if ((int)lane_id() == p) mine = w;
  }
  if (lane_id() < 8) out[((int64_t)lane_id() * n_lines + line) * wpl32 + j] = mine;
}

}  // namespace b2

using namespace b2;

extern "C" {

const char* b2_version(void) { return "bitnn_b200 0.1 (sm_100a)"; }
int64_t b2_launch_count(void) { return g_launches.load(); }

int b2_pack_lines_f32(const float* lines, int64_t n_lines, int64_t bits, uint64_t* out, void* stream) {
  if (n_lines < 0 || bits < 1) return B2_EINVAL;
  int64_t wpl32 = 2 * wpl64(bits);
  int64_t warps = n_lines * wpl32;
  if (!warps) return 0;
  k_pack_lines_f32<<<(unsigned)cdiv(warps, 8), 256, 0, S(stream)>>>(lines, n_lines, bits, wpl32, (uint32_t*)out);
  return launched();
}

int b2_unpack_lines_f32(const uint64_t* words, int64_t n_lines, int64_t bits, float* out, void* stream) {
  if (n_lines < 0 || bits < 1) return B2_EINVAL;
  int64_t n = n_lines * bits;
  if (!n) return 0;
  k_unpack_lines_f32<<<(unsigned)cdiv(n, 256), 256, 0, S(stream)>>>((const uint32_t*)words, n_lines, bits,
                                                                    2 * wpl64(bits), out);
  return launched();
}

int b2_pack_byte_planes(const uint8_t* lines, int64_t n_lines, int64_t bits, uint64_t* out, void* stream) {
  if (n_lines < 0 || bits < 1) return B2_EINVAL;
  int64_t wpl32 = 2 * wpl64(bits);
  int64_t warps = n_lines * wpl32;
  if (!warps) return 0;
  k_pack_byte_planes<<<(unsigned)cdiv(warps, 8), 256, 0, S(stream)>>>(lines, n_lines, bits, wpl32, (uint32_t*)out);
  return launched();
}

}  // extern "C"
