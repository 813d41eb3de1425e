// Kernel launches of the block path: cudaLaunchKernelEx with programmatic
// stream serialization (PDL; see pdl_wait / pdl_trigger in dpb_common.cuh), so
// a kernel's launch and local prologue overlap its predecessor's tail, also
// inside CUDA graphs.  DPB_NO_PDL=1 launches without the attribute.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
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

inline bool pdl_enabled() {
  static const bool on = std::getenv("DPB_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                   Args&&... args) {
  if (current_cat() >= 0 && (skip_mask() >> current_cat() & 1)) return;
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
}

}  // namespace dpb
