// Pipe-throughput microbenchmarks for the binary GEMM design decision
// (SURVEY.md §7.3): POPC on CUDA cores vs legacy mma.sync IMMA (s8, u8)
// vs mma.sync .b1 (emulated on sm_100a).  Prints one JSON line per test.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

// 32 independent popc per iteration; operands rotate so nothing hoists.
__global__ void k_popc(const uint32_t* in, uint32_t* out) {
  uint32_t a[8], b[4], acc[8] = {0};
  for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 1023];
  for (int j = 0; j < 4; ++j) b[j] = in[(threadIdx.x + 17 * j + 3) & 1023];
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i] += __popc(a[i] ^ b[j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = __funnelshift_l(b[j], b[j], 1);
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// pure POPC chain without the xor (upper bound of the POPC pipe)
__global__ void k_popc_raw(const uint32_t* in, uint32_t* out) {
  uint32_t a[16], acc[4] = {0};
  for (int i = 0; i < 16; ++i) a[i] = in[(threadIdx.x + i) & 1023];
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i & 3] += __popc(a[i]);
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] += 0x9e3779b9u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

template <int KIND>
__device__ __forceinline__ void mma_op(int* c, const uint32_t* a, const uint32_t* b) {
  if constexpr (KIND == 0) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  } else if constexpr (KIND == 1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  } else if constexpr (KIND == 2) {
    asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  } else if constexpr (KIND == 3) {
    asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  } else {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
}

template <int KIND>
__global__ void k_mma(const uint32_t* in, int* out) {
  uint32_t a[4], b[8][2];
  int c[8][4] = {};
  for (int i = 0; i < 4; ++i) a[i] = in[(threadIdx.x * 4 + i) & 1023];
  for (int j = 0; j < 8; ++j) { b[j][0] = in[(threadIdx.x + j) & 1023]; b[j][1] = in[(threadIdx.x + 7 * j) & 1023]; }
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) mma_op<KIND>(c[j], a, b[j]);
  }
  int s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  uint32_t *in; int *out;
  CK(cudaMalloc(&in, 4096 * 4)); CK(cudaMalloc(&out, 1 << 26));
  uint32_t h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 0x9e3779b9u * (i + 1);
  CK(cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  auto run = [&](const char* name, auto launch, double ops_per_thread, const char* unit) {
    for (int w = 0; w < 2; ++w) launch();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double ops = ops_per_thread * threads * (double)blocks * reps;
    double per_s = ops / (ms * 1e-3);
    printf("{\"test\": \"%s\", \"ms\": %.3f, \"rate\": %.4e, \"unit\": \"%s\", \"per_sm_per_clk_at_max\": %.2f, \"err\": \"%s\"}\n",
           name, ms / reps, per_s, unit, per_s / sms / (clk_khz * 1e3), cudaGetErrorString(err));
  };
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, sms, clk_khz);
  run("popc_xor (32 xor+popc / thread-iter)", [&] { k_popc<<<blocks, threads>>>(in, (uint32_t*)out); }, 32.0 * ITERS, "popc/s");
  run("popc_raw", [&] { k_popc_raw<<<blocks, threads>>>(in, (uint32_t*)out); }, 16.0 * ITERS, "popc/s");
  // per warp MMA: m16n8k32 = 4096 MAC; per thread share = 4096/32
  run("imma_s8_m16n8k32", [&] { k_mma<0><<<blocks, threads>>>(in, out); }, (ITERS / 8) * 8 * 4096.0 / 32, "MAC/s");
  run("imma_u8s8_m16n8k32", [&] { k_mma<1><<<blocks, threads>>>(in, out); }, (ITERS / 8) * 8 * 4096.0 / 32, "MAC/s");
  run("bmma_and_m16n8k256", [&] { k_mma<2><<<blocks, threads>>>(in, out); }, (ITERS / 8) * 8 * 32768.0 / 32, "bitMAC/s");
  run("bmma_xor_m16n8k256", [&] { k_mma<3><<<blocks, threads>>>(in, out); }, (ITERS / 8) * 8 * 32768.0 / 32, "bitMAC/s");
  run("hmma_bf16_m16n8k16", [&] { k_mma<4><<<blocks, threads>>>(in, out); }, (ITERS / 8) * 8 * 2048.0 / 32, "MAC/s");
  return 0;
}
