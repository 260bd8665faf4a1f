// tcgen05.mma kind::mxf4 (block-scaled packed e2m1, unit scales) issue rate
// on B200 with both operands in shared memory (the only form the kind
// allows), against kind::i8 with A in TMEM: M=128, N in {128, 256}.
// Variant W: 8 other warps stream 16-byte shared-memory stores during the
// loop (the A producers' writes of a kernel that stages A in shared memory),
// to see whether the 128 B/clk shared-memory port caps the tensor rate.
// Also checks the ±1 encoding: with A = B = +1.0 (0x2 nibbles) every
// accumulator must equal K.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
// block-scaled: a/b format E2M1 (=1 for kind::mxf4), scale format UE8M0, K64
__host__ __device__ constexpr uint32_t idesc_mxf4(int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}

// K-major, no swizzle: 8-row x 16-byte core matrices, SBO = 128 B between
// 8-row groups, LBO = K-plane stride (the padded-row conv's band layout)
__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// K-major, 64-byte swizzle: 8-row x 64-byte atoms (SBO = 512)
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (32ull << 32) | (1ull << 46) | (4ull << 61);
}

template <int N, int KIND, int W>  // W: 0 idle, 1 shared-memory stores, 2 TMEM loads (8 warps); KIND 0: i8 (A tmem), 1: mxf4 SS, 2: mxf4 SS with A no-swizzle,
                                    // 3: mxf4 TS (A in TMEM, B no-swizzle shifted by i % 7 rows)
__global__ void k(int iters, long long* clk, float* check) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  __shared__ unsigned long long stores;
  const int warp = threadIdx.x >> 5;
  uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  sbase = (sbase + 1023) & ~1023u;
  uint8_t* sgen = sm + (sbase - (uint32_t)__cvta_generic_to_shared(sm));
  // operands: every byte 0x22 (two +1.0 e2m1 nibbles) / int8 +1
  // RANDOM_OPS: random +-1 operands (e2m1 0x2 / 0xA nibbles, int8 +-1) instead of all +1
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) {
#ifdef RANDOM_OPS
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    sgen[i] = KIND ? (uint8_t)(((h & 1) ? 0x02 : 0x0A) | ((h & 2) ? 0x20 : 0xA0)) : (uint8_t)((h & 1) ? 0x01 : 0xFF);
#else
    sgen[i] = KIND ? 0x22 : 0x01;
#endif
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
    stores = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  // scale factors: columns 256..263 of every lane = 0x7F (2^0) bytes; A-in-TMEM
  // for i8: columns 300.. = 0x01 bytes
  if (warp < 4) {
    const uint32_t lane_base = tm + ((uint32_t)(warp * 32) << 16);
    uint32_t v = 0x7F7F7F7Fu;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + 256 + c), "r"(v));
    uint32_t one = KIND == 3 ? 0x22222222u : 0x01010101u;  // int8 +1 / two e2m1 +1.0 nibbles
    for (int c = 0; c < 32; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + 300 + c), "r"(one));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t bd = desc(sbase + (i & 3) * 32);
      if (KIND == 0) {
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(
                         tm), "r"(tm + 300 + (i & 3) * 8), "l"(bd), "r"(idesc_i8(N)), "r"(i));
      } else if (KIND == 5 || KIND == 8) {
        // TS with a swizzled B: 5 = SW128 (K steps of 32 B in a 128-B row), 8 = SW64
        const uint64_t bds = KIND == 5 ? desc(sbase + 32768 + (i & 3) * 32) : desc_sw64(sbase + 32768 + (i & 1) * 32);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0; "
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;}" ::"r"(tm),
            "r"(tm + 300 + (i & 3) * 8), "l"(bds), "r"(idesc_mxf4(N)), "r"(i), "r"(tm + 256), "r"(tm + 260));
      } else if (KIND >= 4) {
        // 4: A SW128, B no-swizzle shifted by i % 7 rows; 6: A no-swizzle, unshifted; 7: A SW64, B SW128
        uint64_t ad = desc(sbase + 32768 + (i & 3) * 32), bx = bd;
        if (KIND == 4) bx = desc_noswz(sbase + 49152 + (i % 7) * 16, 4096, 128);
        if (KIND == 6) ad = desc_noswz(sbase + 32768 + (i & 1) * 2048, 2048, 128);
        if (KIND == 7) ad = desc_sw64(sbase + 32768 + (i & 1) * 32);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0; "
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;}" ::"r"(tm),
            "l"(ad), "l"(bx), "r"(idesc_mxf4(N)), "r"(i), "r"(tm + 256), "r"(tm + 260));
      } else if (KIND == 3) {
        // A (M = 128 rows) from TMEM, 8 columns per K=64; B rows 16 B apart per K plane, shifted
        const uint64_t bdn = desc_noswz(sbase + 32768 + (i % 7) * 16, 4096, 128);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0; "
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;}" ::"r"(tm),
            "r"(tm + 300 + (i & 3) * 8), "l"(bdn), "r"(idesc_mxf4(N)), "r"(i), "r"(tm + 256), "r"(tm + 260));
      } else {
        // KIND 2: A rows 16 B apart per K plane (planes 2048 B apart), shifted by i % 7 rows
        const uint64_t ad = KIND == 2 ? desc_noswz(sbase + 32768 + (i % 7) * 16, 2048, 128)
                                      : desc(sbase + 32768 + (i & 3) * 32);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0; "
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;}" ::"r"(tm),
            "l"(ad), "l"(bd), "r"(idesc_mxf4(N)), "r"(i), "r"(tm + 256), "r"(tm + 260));
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
    stop = 1;
  } else if (W == 2 && warp >= 4) {
    // 8 warps streaming tcgen05.ld 32x32b.x32 from columns 128..255 (the MMAs write 0..N-1 <= 255:
    // use 384.. for N = 256)
    const uint32_t src = tm + ((uint32_t)((warp & 3) * 32) << 16) + (N == 256 ? 384 : 128) + ((warp >> 2) & 1) * 32;
    unsigned n = 0;
    uint32_t acc = 0;
    while (!stop) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
          "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
            "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
            "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(src));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j];
      ++n;
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(&stores, (unsigned long long)n * 32 * 32 * 4 + (acc == 12345u));
  } else if (W == 1 && warp >= 4) {
    // 8 warps x 32 lanes x 16 B stores into a region the MMAs do not read
    uint4* dst = reinterpret_cast<uint4*>(sgen + 96 * 1024) + ((warp - 4) * 32 + (threadIdx.x & 31));
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    unsigned n = 0;
    while (!stop) {
#pragma unroll
      for (int r = 0; r < 16; ++r) dst[(r & 3) * 256] = v, v.x += 1;
      ++n;
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(&stores, (unsigned long long)n * 16 * 32 * 16);  // bytes by this warp
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4 && blockIdx.x == 0) {  // accumulator check: lane = row, first 8 columns
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    check[threadIdx.x] = KIND ? __uint_as_float(v[0]) : (float)(int)v[0];
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) check[128] = (float)stores;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int KIND, int W>
void run(long long* d, float* chk) {
  const int iters = 20000;
  auto kern = k<N, KIND, W>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  kern<<<148, W ? 384 : 128, 200 * 1024>>>(iters, d, chk);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  float h[129];
  cudaMemcpy(h, chk, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += c[i];
  avg /= 148;
  const int kk = KIND ? 64 : 32;
  double macs = (double)iters * 128 * N * kk;
  printf("{\"mma\": \"%s M=128 N=%d K=%d\", \"smem_store_traffic\": %d, \"clk_per_mma\": %.1f, \"mac_per_clk_per_sm\": %.0f, "
         "\"acc_row0\": %.1f, \"acc_row127\": %.1f, \"expect\": %d, \"store_B_per_clk\": %.1f, \"err\": \"%s\"}\n",
         KIND == 4 ? "mxf4 SS, A SW128, B no-swizzle" : KIND == 5 ? "mxf4 TS, B SW128" :
         KIND == 6 ? "mxf4 SS, A no-swizzle aligned" : KIND == 7 ? "mxf4 SS, A SW64" : KIND == 8 ? "mxf4 TS, B SW64" :
         KIND == 3 ? "mxf4 TS, A in TMEM, B no-swizzle" : KIND == 2 ? "mxf4 SS, A no-swizzle" : (KIND ? "mxf4 SS" : "i8 TS"), N, kk, (int)W, avg / iters, macs / avg, h[0], h[127], iters * kk, h[128] / avg,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  float* chk;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&chk, 129 * 4);
  run<128, 0, 0>(d, chk);
  run<256, 0, 0>(d, chk);
  run<128, 1, 0>(d, chk);
  run<256, 1, 0>(d, chk);
  run<128, 1, 1>(d, chk);
  run<256, 1, 1>(d, chk);
  run<128, 0, 1>(d, chk);
  run<128, 2, 0>(d, chk);
  run<256, 2, 0>(d, chk);
  run<128, 3, 0>(d, chk);
  run<256, 3, 0>(d, chk);
  run<128, 3, 1>(d, chk);
  run<128, 2, 1>(d, chk);
  run<128, 1, 2>(d, chk);
  run<128, 6, 2>(d, chk);
  run<128, 5, 2>(d, chk);
  run<256, 1, 2>(d, chk);
  run<256, 5, 2>(d, chk);
  for (int pass = 0; pass < 1; ++pass) {
    run<128, 4, 0>(d, chk);
    run<256, 4, 0>(d, chk);
    run<128, 5, 0>(d, chk);
    run<256, 5, 0>(d, chk);
    run<128, 6, 0>(d, chk);
    run<128, 7, 0>(d, chk);
    run<128, 8, 0>(d, chk);
    run<128, 4, 1>(d, chk);
    run<128, 5, 1>(d, chk);
    run<128, 7, 1>(d, chk);
  }
  return 0;
}
