// Kernel launches of the block path: cudaLaunchKernelEx with programmatic
// stream serialization (PDL; see pdl_wait / pdl_trigger in dpb_common.cuh), so
// a kernel's launch and local prologue overlap its predecessor's tail, also
// inside CUDA graphs.  DPB_NO_PDL=1 launches without the attribute.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_set>
#include <utility>

namespace dpb {

// Debugging aid for what-if timing: DPB_SKIP_MASK=<bitmask over KernelCat>
// drops every launch made inside a LaunchScope of those categories (results
// are wrong; bench timing only).
inline int& current_cat() {
  static thread_local int cat = -1;
  return cat;
}
inline int skip_mask() {
  static const int m = std::getenv("DPB_SKIP_MASK") ? std::atoi(std::getenv("DPB_SKIP_MASK")) : 0;
  return m;
}

// Kernels launched by this thread through launch() (the model's step count).
inline int64_t& launch_counter() {
  static thread_local int64_t n = 0;
  return n;
}

inline bool pdl_enabled() {
  static const bool on = std::getenv("DPB_NO_PDL") == nullptr;
  return on;
}

// Shared memory above 48 KB (static + dynamic) needs a per-kernel, per-DEVICE opt-in
// (cudaFuncAttributeMaxDynamicSharedMemorySize).  Applied on first use of a
// kernel on the current device, so handles on several GPUs of one process
// each get it (the attribute does not carry across devices).
inline void ensure_smem_optin(const void* kernel, size_t) {
  // every kernel: static + dynamic shared memory above 48 KB needs it too
  static std::mutex mu;
  static std::unordered_set<uint64_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = reinterpret_cast<uintptr_t>(kernel) * 64 + static_cast<uint64_t>(dev & 63);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return;
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kernel);
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       227 * 1024 - static_cast<int>(fa.sharedSizeBytes));
  done.insert(key);
}

// Makes `device` current for the scope of a C-ABI call and restores the
// caller's device on exit (one handle per GPU; the caller may be on another).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != device) cudaSetDevice(device);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                   Args&&... args) {
  if (current_cat() >= 0 && (skip_mask() >> current_cat() & 1)) return;
  ensure_smem_optin(reinterpret_cast<const void*>(kernel), smem);
  ++launch_counter();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  static const bool dbg_sync = std::getenv("DPB_DEBUG_SYNC") != nullptr;  // debugging aid: fault attribution
  if (dbg_sync) {
    const cudaError_t e = cudaDeviceSynchronize();
    const char* name = nullptr;
    cudaFuncGetName(&name, reinterpret_cast<const void*>(kernel));
    if (std::getenv("DPB_DEBUG_SYNC")[0] == '2') fprintf(stderr, "DPB_DEBUG_SYNC: ok %s\n", name ? name : "?");
    if (e != cudaSuccess) {
      fprintf(stderr, "DPB_DEBUG_SYNC: %s after %s\n", cudaGetErrorString(e), name ? name : "?");
    }
  }
}

// As launch(), as thread-block clusters of `cluster` CTAs.
template <typename... KArgs, typename... Args>
inline void launch_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                           dim3 cluster, Args&&... args) {
  if (current_cat() >= 0 && (skip_mask() >> current_cat() & 1)) return;
  ensure_smem_optin(reinterpret_cast<const void*>(kernel), smem);
  ++launch_counter();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster.x;
  attr[1].val.clusterDim.y = cluster.y;
  attr[1].val.clusterDim.z = cluster.z;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace dpb
