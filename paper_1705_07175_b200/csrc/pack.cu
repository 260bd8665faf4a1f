// Sign-binarize / bit-pack kernels.
//
// One warp builds one 32-bit word with __ballot_sync: lane i owns element
// 32*j + i, so ballot bit i is element i of the word — exactly the
// reference's LSB-first order (_kernels.py:6-9).  Lines are padded to whole
// uint64 words; lanes past the line length vote 0, so padding bits are zero.
#include <stdlib.h>

#include "common.cuh"

namespace b2 {

std::atomic<int64_t> g_launches{0};

// programmatic dependent launch on (1) / off (0); B2_PDL in the environment
// sets the initial value, b2_set_pdl() changes it
static std::atomic<int> g_pdl{-1};
bool pdl_enabled() {
  int v = g_pdl.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("B2_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
    g_pdl.store(v, std::memory_order_relaxed);
  }
  return v != 0;
}

// _kernels.py:43-54 pack_lines: bit = !(x < 0)  (0.0, -0.0 and NaN -> 1).
// HBM-bound (4 B in, 1/8 B out per element).  One warp packs 32 words of one
// line per pass: in round r every lane loads element 32 (j0 + r) + lane
// (a coalesced 128-byte row), the ballot is word j0 + r, and lane r keeps
// it, so the 32 words leave as one coalesced 128-byte store.  The 32 loads
// of a pass are independent (full unroll), keeping enough bytes in flight.
__global__ void __launch_bounds__(256) k_pack_lines_f32(const float* __restrict__ lines, int64_t n_lines,
                                                        int64_t bits, int64_t wpl32, uint32_t* __restrict__ out) {
  pdl_entry();
  const int64_t chunks_per_line = (wpl32 + 31) / 32;
  const int64_t chunks = n_lines * chunks_per_line;
  const int lane = lane_id();
  for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < chunks;
       ch += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t line = ch / chunks_per_line;
    const int64_t j0 = (ch - line * chunks_per_line) * 32;
    const float* src = lines + line * bits;
    float v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int64_t b = (j0 + r) * 32 + lane;
      v[r] = b < bits ? __ldg(src + b) : -1.0f;  // past the line: bit 0 (zero padding)
    }
    uint32_t mine = 0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const uint32_t w = __ballot_sync(0xffffffffu, !(v[r] < 0.0f));
      if (lane == r) mine = w;
    }
    if (j0 + lane < wpl32) out[line * wpl32 + j0 + lane] = mine;
  }
}

// _kernels.py:57-64 unpack_lines
__global__ void k_unpack_lines_f32(const uint32_t* __restrict__ words, int64_t n_lines, int64_t bits, int64_t wpl32,
                                   float* __restrict__ out) {
  pdl_entry();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lines * bits) return;
  int64_t line = i / bits, b = i % bits;
  out[i] = ((words[line * wpl32 + (b >> 5)] >> (b & 31)) & 1u) ? 1.0f : -1.0f;
}

// bit p of each of the 4 bytes of v -> a nibble (byte k -> bit k):
// ((v >> p) & 0x01010101) * 0x01020408 puts byte k's bit at 24 + k with no
// other partial product in bits 24..27.
__device__ __forceinline__ uint32_t plane_nibble(uint32_t v, int p) {
  return (((v >> p) & 0x01010101u) * 0x01020408u) >> 24;
}

// _kernels.py:67-82 pack_byte_planes: uint8 lines -> 8 bit-plane lines.
// One warp handles 512 bytes (16 words) of one line per pass: lane l loads
// bytes [16 l, 16 l + 16) (coalesced 16-byte loads), builds for every
// plane the 16-bit mask of its bytes, and even lanes join their odd
// neighbour's mask into the plane's 32-bit word.
__global__ void __launch_bounds__(256) k_pack_byte_planes(const uint8_t* __restrict__ lines, int64_t n_lines,
                                                          int64_t bits, int64_t wpl32, uint32_t* __restrict__ out) {
  pdl_entry();
  const int64_t chunks_per_line = (wpl32 + 15) / 16;
  const int64_t chunks = n_lines * chunks_per_line;
  const int lane = lane_id();
  for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < chunks;
       ch += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t line = ch / chunks_per_line;
    const int64_t w0 = (ch - line * chunks_per_line) * 16;  // first word of this pass
    const int64_t b0 = w0 * 32 + 16 * lane;                 // this lane's first byte
    const uint8_t* src = lines + line * bits;
    uint4 x = make_uint4(0, 0, 0, 0);
    if (b0 + 16 <= bits && (((uintptr_t)(src + b0)) & 15) == 0) {
      x = __ldg(reinterpret_cast<const uint4*>(src + b0));
    } else {
      uint32_t* xb = reinterpret_cast<uint32_t*>(&x);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (b0 + i < bits) xb[i >> 2] |= (uint32_t)__ldg(src + b0 + i) << (8 * (i & 3));
    }
    const int64_t w = w0 + (lane >> 1);
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const uint32_t m16 = plane_nibble(x.x, p) | plane_nibble(x.y, p) << 4 | plane_nibble(x.z, p) << 8 |
                           plane_nibble(x.w, p) << 12;
      const uint32_t hi = __shfl_down_sync(0xffffffffu, m16, 1);
      if (!(lane & 1) && w < wpl32) out[((int64_t)p * n_lines + line) * wpl32 + w] = m16 | (hi << 16);
    }
  }
}

}  // namespace b2

using namespace b2;

extern "C" {

const char* b2_version(void) { return "bitnn_b200 0.1 (sm_100a)"; }
int64_t b2_launch_count(void) { return g_launches.load(); }
int b2_set_pdl(int on) {
  const int was = pdl_enabled() ? 1 : 0;
  g_pdl.store(on ? 1 : 0, std::memory_order_relaxed);
  return was;
}

int b2_pack_lines_f32(const float* lines, int64_t n_lines, int64_t bits, uint64_t* out, void* stream) {
  if (n_lines < 0 || bits < 1) return B2_EINVAL;
  int64_t wpl32 = 2 * wpl64(bits);
  int64_t chunks = n_lines * cdiv(wpl32, 32);
  if (!chunks) return 0;
  const int64_t blocks = cdiv(chunks, 8) < 148 * 32 ? cdiv(chunks, 8) : 148 * 32;  // grid-stride beyond
  launch_k(k_pack_lines_f32, (unsigned)blocks, 256, 0, S(stream), lines, n_lines, bits, wpl32, (uint32_t*)out);
  return launched();
}

int b2_unpack_lines_f32(const uint64_t* words, int64_t n_lines, int64_t bits, float* out, void* stream) {
  if (n_lines < 0 || bits < 1) return B2_EINVAL;
  int64_t n = n_lines * bits;
  if (!n) return 0;
  launch_k(k_unpack_lines_f32, (unsigned)cdiv(n, 256), 256, 0, S(stream), (const uint32_t*)words, n_lines, bits,
                                                                    2 * wpl64(bits), out);
  return launched();
}

int b2_pack_byte_planes(const uint8_t* lines, int64_t n_lines, int64_t bits, uint64_t* out, void* stream) {
  if (n_lines < 0 || bits < 1) return B2_EINVAL;
  int64_t wpl32 = 2 * wpl64(bits);
  int64_t chunks = n_lines * cdiv(wpl32, 16);
  if (!chunks) return 0;
  const int64_t blocks = cdiv(chunks, 8) < 148 * 32 ? cdiv(chunks, 8) : 148 * 32;  // grid-stride beyond
  launch_k(k_pack_byte_planes, (unsigned)blocks, 256, 0, S(stream), lines, n_lines, bits, wpl32, (uint32_t*)out);
  return launched();
}

}  // extern "C"
