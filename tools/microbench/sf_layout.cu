// Probe: the TMEM layout of kind::mxf4 block scale factors (SFA at column
// 256, SFB at 260; A in TMEM, all +1; B no-swizzle all +1).  Mode 0 varies
// SFB bytes per lane, mode 1 SFA bytes per lane (exponent = lane % 5 in byte
// 0, 0 in byte 1, 7 in bytes 2-3); D = 32 (2^ea0+eb0 + 2^ea1+eb1) tells which
// lane / byte each row / K block reads.
// One CTA: A words (16 per lane, columns 300..315) and a no-swizzle K-major B
// (128 rows, two 16-byte K planes 2048 B apart) come from the host, one
// M = 128, N = 128, K = 64 MMA runs with unit scales, and D (fp32) goes back.
// tools/microbench/ts_layout.py decides which nibble -> K mapping matches.
#include <cstdint>
#include <cstdio>
#include <vector>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr uint32_t idesc_mxf4(int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}
__device__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void k(const uint32_t* aw, const uint8_t* bb, float* d, int mode) {
  __shared__ __align__(1024) uint8_t sb[4096];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += 128) sb[i] = bb[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const uint32_t lb = tm + ((uint32_t)(warp * 32) << 16);
  const int m = warp * 32 + lane;
  // mode bit 1: vary SFA (columns 256..259) else SFB (260..263); bit 0:
  // byte 0 exponent = 4 (column - base) + lane / 32, else lane % 32 (byte 1: 0)
  for (int c = 0; c < 16; ++c) {
    uint32_t sf = 0x7F7F7F7Fu;
    const int base = (mode & 2) ? 0 : 4;
    if (c >= base && c < base + 4) {
      const uint32_t e = (mode & 1) ? (uint32_t)(4 * (c - base) + m / 32) : (uint32_t)(m % 32);
      sf = (127u + e) | (127u << 8) | (127u << 16) | (127u << 24);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lb + 256 + c), "r"(sf));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lb + 300 + c), "r"(aw[m * 16 + c]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint64_t bd = desc_noswz(smem_u32(sb), 2048, 128);
    asm volatile(
        "{.reg .pred p; setp.ne.b32 p, 0, 0; "
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%4], [%5], p;}" ::"r"(tm),
        "r"(tm + 300), "l"(bd), "r"(idesc_mxf4(128)), "r"(tm + 256), "r"(tm + 260));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile(
      "{.reg .pred P1; LAB_WAIT: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @P1 bra DONE; bra LAB_WAIT; DONE: }" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < 128; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(lb + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    d[m * 128 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main(int argc, char** argv) {
  const char* out = argc > 1 ? argv[1] : "ts_layout.bin";
  std::mt19937 rng(7);
  std::vector<uint32_t> aw(128 * 16);
  std::vector<uint8_t> bb(4096, 0);
  const uint8_t code[3] = {0x0, 0x2, 0xA};  // 0, +1, -1 (e2m1)
  (void)code;
  for (int m = 0; m < 128; ++m)
    for (int c = 0; c < 16; ++c) aw[m * 16 + c] = c < 8 ? 0x22222222u : 0u;
  for (int p = 0; p < 2; ++p)
    for (int n = 0; n < 128; ++n)
      for (int b = 0; b < 16; ++b) bb[p * 2048 + n * 16 + b] = 0x22;
  uint32_t* daw;
  uint8_t* dbb;
  float* dd;
  cudaMalloc(&daw, aw.size() * 4);
  cudaMalloc(&dbb, bb.size());
  cudaMalloc(&dd, 128 * 128 * 4);
  cudaMemcpy(daw, aw.data(), aw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dbb, bb.data(), bb.size(), cudaMemcpyHostToDevice);
  FILE* f = fopen(out, "wb");
  for (int mode = 0; mode < 4; ++mode) {
    k<<<1, 128>>>(daw, dbb, dd, mode);
    cudaDeviceSynchronize();
    std::vector<float> d(128 * 128);
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    fwrite(d.data(), 4, d.size(), f);
  }
  fclose(f);
  printf("%s %s\n", out, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
