// Raw tcgen05.mma kind::i8 issue rate on B200 (one CTA per SM, one thread
// issuing back-to-back MMAs on resident operands, no data movement):
// M=128, N in {64,128,256}, A from TMEM (TS) or shared memory (SS).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

template <int N, bool TS, int CE>
__global__ void k(int iters, long long* clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t dummy[2];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&dummy[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&dummy[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  sbase = (sbase + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (CE && i % CE == 0 && i)  // commit every CE MMAs (two barriers, like the GEMM's B and A rings)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
                     "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&dummy[0])), "r"((uint32_t)__cvta_generic_to_shared(&dummy[1])));
      const uint64_t bd = desc(sbase + (i & 3) * 32);
      if (TS) {
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(
                         tm), "r"(tm + 256 + (i & 3) * 8), "l"(bd), "r"(idesc(N)), "r"(i));
      } else {
        const uint64_t ad = desc(sbase + 65536 + (i & 3) * 32);
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::"r"(
                         tm), "l"(ad), "l"(bd), "r"(idesc(N)), "r"(i));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(done)
                   : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
    long long t1 = clock64();
    clk[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, bool TS, int CE = 0>
void run(long long* d) {
  const int iters = 20000;
  auto kern = k<N, TS, CE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  kern<<<148, 128, 140 * 1024>>>(iters, d);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  double macs = (double)iters * 128 * N * 32;
  printf("{\"mma\": \"i8 M=128 N=%d K=32 %s\", \"commit_every\": %d, \"clk_per_mma\": %.1f, \"mac_per_clk_per_sm\": %.0f, \"err\": \"%s\"}\n", N,
         TS ? "A:tmem" : "A:smem", CE, avg / iters, macs / avg, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  run<64, true>(d);
  run<128, true>(d);
  run<256, true>(d);
  run<64, false>(d);
  run<128, false>(d);
  run<256, false>(d);
  run<128, true, 4>(d);
  run<128, true, 8>(d);
  run<256, true, 4>(d);
  run<256, true, 8>(d);
  return 0;
}
