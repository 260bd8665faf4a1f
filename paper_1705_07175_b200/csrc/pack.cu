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

// ---------------------------------------------------------------- TMA-fed variants
// Both packing kernels are HBM streams; with the bytes in flight held in
// registers their occupancy (and so the bytes in flight) is register-bound.
// These variants stage each warp's input through a 3-slot shared-memory ring
// filled by 1-D bulk copies (cp.async.bulk, completion on an mbarrier): the
// copies of the next two chunks are in flight while the warp packs the
// current one from shared memory.  Eligible when every chunk is a 16-byte
// multiple at a 16-byte aligned address (lines of bits % 4 == 0 floats /
// bits % 16 == 0 bytes); other shapes keep the kernels above.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(smem_addr(bar)), "r"(parity)
                 : "memory");
  } while (!done);
}

constexpr int PK_WARPS = 8, PK_SLOTS = 3;

// chunk = 1024 floats (32 words) of one line, as k_pack_lines_f32
__global__ void __launch_bounds__(32 * PK_WARPS) k_pack_lines_f32_tma(const float* __restrict__ lines, int64_t n_lines,
                                                                       int64_t bits, int64_t wpl32,
                                                                       uint32_t* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t pk_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* ring = reinterpret_cast<float*>(pk_smem) + warp * PK_SLOTS * 1024;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pk_smem + PK_WARPS * PK_SLOTS * 4096) + warp * PK_SLOTS;
  if (lane == 0)
    for (int i = 0; i < PK_SLOTS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  pdl_entry();
  const uint32_t cpl = (uint32_t)((wpl32 + 31) / 32);  // chunks per line
  const uint32_t chunks = (uint32_t)(n_lines * cpl);
  const uint32_t step = gridDim.x * PK_WARPS;
  const uint32_t c0 = blockIdx.x * PK_WARPS + warp;
  auto issue = [&](uint32_t c, int slot) {
    if (c >= chunks) return;
    const uint32_t line = c / cpl, j = c - line * cpl;
    const int64_t e0 = (int64_t)j * 1024;
    const int64_t n = bits - e0 < 1024 ? bits - e0 : 1024;
    bulk_g2s(ring + slot * 1024, lines + line * bits + e0, (uint32_t)(n * 4), &bars[slot]);
  };
  if (lane == 0) {
    issue(c0, 0);
    issue(c0 + step, 1);
  }
  int slot = 0;
  uint32_t ph = 0;
  for (uint32_t c = c0; c < chunks; c += step) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the warp's reads of that slot came first
      issue(c + 2 * step, slot == 0 ? PK_SLOTS - 1 : slot - 1);
    }
    const uint32_t line = c / cpl, j = c - line * cpl;
    const int64_t e0 = (int64_t)j * 1024;
    const int n = (int)(bits - e0 < 1024 ? bits - e0 : 1024);
    bar_wait(&bars[slot], ph);
    const float* v = ring + slot * 1024;
    uint32_t mine = 0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int e = r * 32 + lane;
      const uint32_t w = __ballot_sync(0xffffffffu, e < n && !(v[e] < 0.0f));
      if (lane == r) mine = w;
    }
    if (j * 32 + lane < wpl32) out[line * wpl32 + j * 32 + lane] = mine;
    __syncwarp();
    if (++slot == PK_SLOTS) slot = 0, ph ^= 1;
  }
}

// The same transpose on the word's two 32-bit halves (lo = bytes 0-3): the
// 7- and 14-bit delta swaps stay inside a half, the 28-bit one swaps nibbles
// between the halves
__device__ __forceinline__ void transpose8_32(uint32_t& lo, uint32_t& hi) {
  uint32_t t = (lo ^ (lo >> 7)) & 0x00AA00AAu;
  lo ^= t ^ (t << 7);
  t = (hi ^ (hi >> 7)) & 0x00AA00AAu;
  hi ^= t ^ (t << 7);
  t = (lo ^ (lo >> 14)) & 0x0000CCCCu;
  lo ^= t ^ (t << 14);
  t = (hi ^ (hi >> 14)) & 0x0000CCCCu;
  hi ^= t ^ (t << 14);
  t = (lo ^ (hi << 4)) & 0xF0F0F0F0u;
  lo ^= t;
  hi ^= t >> 4;
}

// 8x8 bit transpose of a 64-bit word (row i = byte i): byte p of the result
// holds bit p of every input byte (Hacker's Delight delta swaps)
__device__ __forceinline__ uint64_t transpose8(uint64_t x) {
  uint64_t t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
  x = x ^ t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
  x = x ^ t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
  return x ^ t ^ (t << 28);
}

// chunk = LB whole lines (LB = 4096 / bits, lines of at most 4096 bytes): one
// bulk copy per chunk (small copies are TMA-issue-bound), then per line and
// 512-byte segment lane l packs bytes [16 l, 16 l + 16) by two 8x8 bit
// transposes; even lanes join their odd neighbour's 16 bits into the word
constexpr int PK_BYTES_SLOT = 4096;
__global__ void __launch_bounds__(32 * PK_WARPS) k_pack_byte_planes_tma(const uint8_t* __restrict__ lines,
                                                                         int64_t n_lines, int64_t bits, int64_t wpl32,
                                                                         uint32_t* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t pk_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = pk_smem + warp * PK_SLOTS * PK_BYTES_SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(pk_smem + PK_WARPS * PK_SLOTS * PK_BYTES_SLOT) + warp * PK_SLOTS;
  if (lane == 0)
    for (int i = 0; i < PK_SLOTS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  pdl_entry();
  const int lb = (int)(PK_BYTES_SLOT / bits);  // lines per chunk
  const int bw = (int)bits;
  const uint32_t chunks = (uint32_t)((n_lines + lb - 1) / lb);
  const uint32_t step = gridDim.x * PK_WARPS;
  const uint32_t c0 = blockIdx.x * PK_WARPS + warp;
  auto issue = [&](uint32_t c, int slot) {
    if (c >= chunks) return;
    const int64_t l0 = (int64_t)c * lb;
    const int64_t nl = n_lines - l0 < lb ? n_lines - l0 : lb;
    bulk_g2s(ring + slot * PK_BYTES_SLOT, lines + l0 * bits, (uint32_t)(nl * bits), &bars[slot]);
  };
  if (lane == 0) {
    issue(c0, 0);
    issue(c0 + step, 1);
  }
  int slot = 0;
  uint32_t ph = 0;
  for (uint32_t c = c0; c < chunks; c += step) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the warp's reads of that slot came first
      issue(c + 2 * step, slot == 0 ? PK_SLOTS - 1 : slot - 1);
    }
    const int64_t l0 = (int64_t)c * lb;
    const int nl = (int)(n_lines - l0 < lb ? n_lines - l0 : lb);
    bar_wait(&bars[slot], ph);
    const uint8_t* buf = ring + slot * PK_BYTES_SLOT;
    for (int li = 0; li < nl; ++li) {
      const int64_t line = l0 + li;
      for (int b0 = 0; b0 < bw; b0 += 512) {
        const int n = bw - b0 < 512 ? bw - b0 : 512;  // valid bytes of this segment
        uint4 x = make_uint4(0, 0, 0, 0);
        if (16 * lane < n) x = *reinterpret_cast<const uint4*>(buf + li * bw + b0 + 16 * lane);  // n % 16 == 0
        transpose8_32(x.x, x.y);
        transpose8_32(x.z, x.w);
        const int64_t w = b0 / 32 + (lane >> 1);
        uint32_t* o = out + line * wpl32 + w;
        const int64_t pstride = n_lines * wpl32;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          // [byte p of bytes 0-7, byte p of bytes 8-15] of this lane, then the
          // odd neighbour's two bytes above them: the plane's 32-bit word
          const uint32_t a = p < 4 ? x.x : x.y, b = p < 4 ? x.z : x.w;
          const uint32_t m16 = __byte_perm(a, b, (uint32_t)((p & 3) | ((4 + (p & 3)) << 4)));
          const uint32_t hi = __shfl_down_sync(0xffffffffu, m16, 1);
          if (!(lane & 1) && w < wpl32) o[p * pstride] = __byte_perm(m16, hi, 0x5410);
        }
      }
    }
    __syncwarp();
    if (++slot == PK_SLOTS) slot = 0, ph ^= 1;
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
  if (bits % 4 == 0 && (reinterpret_cast<uintptr_t>(lines) & 15) == 0 && chunks < (int64_t)1 << 31) {
    static std::atomic<uint64_t> attr{0};
    const int smem = PK_WARPS * PK_SLOTS * (4096 + 8);
    smem_optin(k_pack_lines_f32_tma, smem, attr);
    const int64_t blocks = cdiv(chunks, PK_WARPS) < 148 * 2 ? cdiv(chunks, PK_WARPS) : 148 * 2;
    launch_k(k_pack_lines_f32_tma, (unsigned)blocks, 32 * PK_WARPS, smem, S(stream), lines, n_lines, bits, wpl32,
             (uint32_t*)out);
    return launched();
  }
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
  if (bits % 16 == 0 && bits <= PK_BYTES_SLOT && (reinterpret_cast<uintptr_t>(lines) & 15) == 0 &&
      n_lines < (int64_t)1 << 31) {
    static std::atomic<uint64_t> attr{0};
    const int smem = PK_WARPS * PK_SLOTS * (PK_BYTES_SLOT + 8);
    smem_optin(k_pack_byte_planes_tma, smem, attr);
    const int64_t tchunks = cdiv(n_lines, PK_BYTES_SLOT / bits);
    const int64_t blocks = cdiv(tchunks, PK_WARPS) < 148 * 2 ? cdiv(tchunks, PK_WARPS) : 148 * 2;
    launch_k(k_pack_byte_planes_tma, (unsigned)blocks, 32 * PK_WARPS, smem, S(stream), lines, n_lines, bits, wpl32,
             (uint32_t*)out);
    return launched();
  }
  const int64_t blocks = cdiv(chunks, 8) < 148 * 32 ? cdiv(chunks, 8) : 148 * 32;  // grid-stride beyond
  launch_k(k_pack_byte_planes, (unsigned)blocks, 256, 0, S(stream), lines, n_lines, bits, wpl32, (uint32_t*)out);
  return launched();
}

}  // extern "C"
