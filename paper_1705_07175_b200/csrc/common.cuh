// Shared helpers for the sm_100a kernels of the binary forward pass.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>

#include "../../include/bitnn_b200.h"

namespace b2 {

extern std::atomic<int64_t> g_launches;

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Count one launch and report its configuration error (if any).
inline int launched() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : static_cast<int>(e);
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch: every kernel is launched with
// programmatic stream serialization, so its launch, CTA placement and
// prologue overlap the tail of the kernel before it on the stream (the
// per-layer chain of a forward pass at batch 1 is mostly that latency).
// Each kernel calls griddepcontrol.wait before it touches global memory the
// previous kernel may read or write, and releases its own dependents right
// after.  B2_PDL=0 launches plainly (both instructions are then no-ops).
bool pdl_enabled();
// `cluster` > 1: thread-block clusters of that many CTAs along x
template <typename... KArgs, typename... Args>
inline void launch_kc(int cluster, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args... args) {
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = (unsigned)cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n++].val.clusterDim.z = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, kern, args...);  // errors surface through launched()
}
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  launch_kc(1, kern, grid, block, smem, st, args...);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() {
  pdl_wait();
  pdl_trigger();
}

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device,
// once per (kernel, device): the attribute is per device, and one process
// may drive several GPUs.  `done` is the caller's per-kernel static bitmask.
template <typename K>
inline void smem_optin(K kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_relaxed) & bit) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_relaxed);
}
inline int64_t wpl64(int64_t bits) { return (bits + 63) >> 6; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Bits [lo, lo+len) (len <= 64) of a packed line, LSB-first.
__device__ __forceinline__ uint64_t get_bits64(const uint64_t* line, int64_t lo, int len) {
  if (len <= 0) return 0;
  int64_t w = lo >> 6;
  int sh = (int)(lo & 63);
  uint64_t v = line[w] >> sh;
  if (sh && sh + len > 64) v |= line[w + 1] << (64 - sh);
  if (len < 64) v &= (1ULL << len) - 1ULL;
  return v;
}

// threshold rule of _kernels.py:261 (int32 clamped form, see include/bitnn_b200.h)
__device__ __forceinline__ bool thr_bit(int32_t v, int32_t t, bool ge) { return ge ? (v >= t) : (v <= t); }

// cp.async with zero fill (src_bytes = 0 -> the destination is zeroed)
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, bool valid) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  int n = valid ? BYTES : 0;
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES), "r"(n));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace b2
