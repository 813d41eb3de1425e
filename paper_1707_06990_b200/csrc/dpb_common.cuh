// Shared device helpers for the dense-block kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dpb {

constexpr float kEps = 1e-5f;       // BatchNormState::eps, ops.hpp:22
constexpr float kMomentum = 0.1f;   // BatchNormState::momentum, ops.hpp:23

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename S>
__device__ __forceinline__ S from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// 1 / sqrt(var + eps) evaluated like the reference: T(1) / std::sqrt(v + eps)
// (ops.hpp:124, :219).  IEEE sqrt and division (no fast-math).
__device__ __forceinline__ float bn_inv(float var) {
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, kEps)));
}

// Per-channel BN forward transform kept in shared memory by the kernels that
// recompute BN+ReLU in their prologue: y = (x - mean) * (gamma*inv) + beta.
struct BnFwd {
  float mean, scale, beta, inv, gamma;
};

// Compact forward BN affine of one channel, y = x * scale + shift with
// scale = gamma*inv, shift = beta - mean*scale: 8 bytes per channel, so the 1x1
// forward can keep a table of every input channel (c up to ~4k) in shared memory.
struct BnAff {
  float scale, shift;
};

// The ReLU mask of the backward pass, act > 0, evaluated with the
// reference's exact float expression gamma * (x - mean) * inv + beta
// (ops.hpp:130, left to right, no contraction) so that, given the same
// stored forward values, the mask is bit-identical to the reference's
// relu_backward predicate (ops.hpp:268-287).
__device__ __forceinline__ bool relu_mask_ref(const BnFwd& b, float x) {
  const float t = __fmul_rn(__fmul_rn(b.gamma, __fsub_rn(x, b.mean)), b.inv);
  return __fadd_rn(t, b.beta) > 0.f;
}

// BN backward coefficients of one channel (ops.hpp:206-243):
//   gx = (gamma*inv) * (g - mg - xhat * mgx),   xhat = (x - mean) * inv
struct BnBwd {
  float mean, inv, ginv, mg, mgx;
};

// Programmatic dependent launch (PDL): every block-path kernel is launched with
// programmatic stream serialization (dpb_launch.h).  A kernel waits for its
// predecessor's completion (griddepcontrol.wait) before its first global read
// of data written by a kernel, then lets its own dependents start launching:
// triggering only after the wait guarantees that, when a kernel starts, every
// kernel but its immediate predecessor has completed.  Both are no-ops for a
// launch without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

}  // namespace dpb
