// The GEMM's MMA-issuer loop in isolation: per stage, wait on two
// (already-completed) mbarriers, tcgen05.fence::after_thread_sync, MMAS
// tcgen05.mma kind::i8 (M=128, A from TMEM), two tcgen05.commit.  Measures
// cycles per MMA for each ingredient toggled.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  uint32_t done;
  do {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(done)
                 : "r"(bar), "r"(par)
                 : "memory");
  } while (!done);
}

__device__ __forceinline__ bool test(uint32_t bar, uint32_t par) {
  uint32_t done;
  asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
               : "=r"(done)
               : "r"(bar), "r"(par)
               : "memory");
  return done;
}

// WAITS: 0 none, 1 two try_waits, 2 one try_wait, 3 one test_wait (spin)
// COMMITS: 0 none, 1 two, 2 one
template <int N, int MMAS, int WAITS, bool FENCE, int COMMITS>
__global__ void k(int stages, long long* clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[4];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);
  const uint32_t b1 = (uint32_t)__cvta_generic_to_shared(&bars[1]);
  const uint32_t c0 = (uint32_t)__cvta_generic_to_shared(&bars[2]);
  const uint32_t c1 = (uint32_t)__cvta_generic_to_shared(&bars[3]);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      if (WAITS == 1) {  // parity 1 of a fresh barrier: completes immediately
        wait(b0, 1);
        wait(b1, 1);
      } else if (WAITS == 2) {
        wait(b0, 1);
      } else if (WAITS == 3) {
        while (!test(b0, 1)) {
        }
      }
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < MMAS; ++k) {
        const uint64_t bd = desc(sbase + (k >> 2) * N * 128 + (k & 3) * 32);
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(
                         tm), "r"(tm + 256 + k * 8), "l"(bd), "r"(idesc(N)), "r"(st | k)
                     : "memory");
      }
      if (COMMITS == 2)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(c0)
                     : "memory");
      if (COMMITS == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
                     "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];" ::"r"(c0),
                     "r"(c1)
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0) : "memory");
    wait(b0, 0);
    long long t1 = clock64();
    clk[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int MMAS, int WAITS, bool FENCE, int COMMITS>
void run(long long* d) {
  const int stages = 4000;
  auto kern = k<N, MMAS, WAITS, FENCE, COMMITS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kern<<<148, 128, 100 * 1024>>>(stages, d);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  printf("{\"N\": %d, \"mmas_per_stage\": %d, \"waits\": %d, \"fence\": %d, \"commits\": %d, \"clk_per_mma\": %.1f, "
         "\"frac_of_peak\": %.3f, \"err\": \"%s\"}\n",
         N, MMAS, WAITS, FENCE, COMMITS, avg / (stages * MMAS), (N / 2.0) / (avg / (stages * MMAS)),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  run<128, 8, 0, false, 0>(d);
  run<128, 8, 1, true, 1>(d);
  run<128, 8, 2, true, 2>(d);
  run<128, 8, 3, true, 2>(d);
  run<128, 8, 2, false, 2>(d);
  run<128, 16, 2, true, 2>(d);
  run<128, 4, 2, true, 2>(d);
  run<128, 4, 3, true, 2>(d);
  run<256, 4, 2, true, 2>(d);
  return 0;
}
