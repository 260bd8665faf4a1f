// Stand-alone check of the tcgen05 kind::i8 binary GEMM against a CPU
// popcount GEMM, plus timing.  Build: make -C tools/tc_probe; run on a B200.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <random>
#include "../../include/bitnn_b200.h"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

// pack=1: b2_tc_dense_bn_pack (threshold acc >= 0, packed bits out), the
// epilogue the conv/dense stages use; pack=0: int32 output.
static int g_pack = 0;

static int run(int64_t M, int64_t N, int64_t K, int reps, bool check_all) {
  int64_t wpl = (K + 63) / 64;
  std::mt19937_64 rng(M * 131 + N * 7 + K);
  std::vector<uint64_t> A(M * wpl), B(N * wpl);
  auto fill = [&](std::vector<uint64_t>& v) {
    for (int64_t r = 0; r < (int64_t)v.size() / wpl; ++r)
      for (int64_t w = 0; w < wpl; ++w) {
        uint64_t x = rng();
        int64_t hi = K - 64 * w;
        if (hi < 64) x &= hi <= 0 ? 0 : ((1ull << hi) - 1);
        v[r * wpl + w] = x;
      }
  };
  fill(A); fill(B);
  uint64_t *dA, *dB; int8_t* dBi; int32_t* dC;
  int64_t kpad = b2_i8_kpad(K);
  CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8));
  CK(cudaMalloc(&dBi, N * kpad)); CK(cudaMalloc(&dC, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0x7f, M * N * 4));
  if (b2_expand_i8(dB, N, wpl, K, 1, dBi, 0)) { printf("expand failed\n"); return 1; }
  int32_t* dT;
  uint8_t* dG;
  uint64_t* dP;
  int64_t owpl = (N + 63) / 64;
  CK(cudaMalloc(&dT, N * 4));
  CK(cudaMalloc(&dG, N));
  CK(cudaMalloc(&dP, M * owpl * 8));
  CK(cudaMemset(dT, 0, N * 4));
  CK(cudaMemset(dG, 1, N));
  b2_thresh th{dT, nullptr, dG};
  auto launch = [&]() {
    return g_pack ? b2_tc_dense_bn_pack(dA, M, dBi, N, wpl, (int)K, th, dP, 0)
                  : b2_tc_bgemm(dA, M, dBi, N, wpl, (int)K, dC, 0);
  };
  int rc = launch();
  if (rc) { printf("launch rc=%d\n", rc); return 1; }
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> C(M * N);
  std::vector<uint64_t> P(M * owpl);
  if (g_pack) CK(cudaMemcpy(P.data(), dP, P.size() * 8, cudaMemcpyDeviceToHost));
  else CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  int64_t bad = 0, checked = 0;
  std::mt19937_64 pick(5);
  int64_t samples = check_all ? M * N : 20000;
  for (int64_t s = 0; s < samples; ++s) {
    int64_t i, j;
    if (check_all) { i = s / N; j = s % N; } else { i = pick() % M; j = pick() % N; }
    int p = 0;
    for (int64_t w = 0; w < wpl; ++w) p += __builtin_popcountll(A[i * wpl + w] ^ B[j * wpl + w]);
    int32_t ref = (int32_t)K - 2 * p;
    ++checked;
    if (g_pack) {
      int bit = (int)((P[i * owpl + j / 64] >> (j % 64)) & 1);
      if (bit != (ref >= 0)) { if (bad < 5) printf("  bit mismatch (%ld,%ld)\n", (long)i, (long)j); ++bad; }
      continue;
    }
    if (C[i * N + j] != ref) { if (bad < 5) printf("  mismatch (%ld,%ld): got %d want %d\n", (long)i, (long)j, C[i * N + j], ref); ++bad; }
  }
  float ms = 0;
  if (reps > 0) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int r = 0; r < 2; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  }
  double tops = ms > 0 ? 2.0 * M * N * K / (ms * 1e-3) / 1e12 : 0;
  printf("{\"pack\": %d, \"M\": %ld, \"N\": %ld, \"K\": %ld, \"checked\": %ld, \"bad\": %ld, \"ms\": %.4f, \"Tbitops\": %.1f}\n",
         g_pack, (long)M, (long)N, (long)K, (long)checked, (long)bad, ms, tops);
  fflush(stdout);
  cudaFree(dA); cudaFree(dB); cudaFree(dBi); cudaFree(dC); cudaFree(dT); cudaFree(dG); cudaFree(dP);
  return bad != 0;
}

int main(int argc, char** argv) {
  if (argc >= 6) g_pack = atoi(argv[5]);
  if (argc >= 4) return run(atoll(argv[1]), atoll(argv[2]), atoll(argv[3]), argc > 4 ? atoi(argv[4]) : 5, false);
  int fails = 0;
  fails += run(128, 128, 128, 0, true);
  fails += run(256, 128, 256, 0, true);
  fails += run(300, 200, 300, 0, true);
  fails += run(1000, 130, 1000, 0, true);
  fails += run(1024, 1024, 1024, 10, false);
  fails += run(4096, 4096, 4096, 10, false);
  fails += run(8192, 8192, 8192, 5, false);
  fails += run(16384, 16384, 16384, 3, false);
  printf("fails=%d\n", fails);
  return fails;
}
