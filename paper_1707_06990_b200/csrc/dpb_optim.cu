// Momentum SGD with weight decay over the flat parameter buffer, and the
// learning-rate schedules (dp/train.hpp:43-70,
// dp/schedule.hpp:46-62).  One fused HBM-bound pass: reads p, g, v and
// writes p, v (20 bytes per parameter).  Each product and sum is rounded on
// its own (__fmul_rn / __fadd_rn, no FMA contraction), so the update is
// bit-identical to the reference's float loop.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "dpb_common.cuh"
#include "dpb_internal.h"
#include "dpb_launch.h"

namespace dpb {
namespace {

__global__ void k_sgd(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ v, int64_t n,
                      float lr, float mu, float wd, int nesterov) {
  pdl_enter();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float pi = p[i];
    const float d = __fadd_rn(g[i], __fmul_rn(wd, pi));        // d = g + wd*p
    const float vn = __fadd_rn(__fmul_rn(mu, v[i]), d);        // v = mu*v + d
    v[i] = vn;
    const float step = nesterov ? __fadd_rn(d, __fmul_rn(mu, vn)) : vn;
    p[i] = __fsub_rn(pi, __fmul_rn(lr, step));                 // p -= lr * step
  }
}

}  // namespace
}  // namespace dpb

using namespace dpb;

extern "C" {

DPB_API int dpb_sgd_step(float* params, const float* grads, float* velocity, int64_t n, double lr,
                         double momentum, double weight_decay, int nesterov, void* stream) {
  if (n < 0) return fail(DPB_SHAPE_ERROR, "negative parameter count");
  if (n == 0) return DPB_OK;
  if (!params || !grads || !velocity) return fail(DPB_CONFIG_ERROR, "null pointer argument");
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 8);
  launch(k_sgd, static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream), params, grads,
         velocity, n, static_cast<float>(lr), static_cast<float>(momentum), static_cast<float>(weight_decay),
         nesterov);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DPB_OK : cuda_fail(e, "sgd launch");
}

DPB_API int dpb_lr_at(int kind, double base_lr, int total_epochs, const int32_t* milestones, int nmilestones,
                      double factor, double floor_lr, int epoch, double* out) {
  if (out == nullptr) return fail(DPB_CONFIG_ERROR, "null output");
  if (epoch < 0 || epoch >= total_epochs)
    return fail(DPB_RANGE_ERROR, "epoch " + std::to_string(epoch) + " outside [0, " +
                                     std::to_string(total_epochs) + ")");
  if (kind == 1) {  // cosine
    const double pi = 3.14159265358979323846;
    *out = floor_lr + (base_lr - floor_lr) / 2.0 *
                          (std::cos(pi * static_cast<double>(epoch) / total_epochs) + 1.0);
    return DPB_OK;
  }
  double lr = base_lr;
  for (int i = 0; i < nmilestones; ++i)
    if (epoch >= milestones[i]) lr *= factor;
  *out = lr;
  return DPB_OK;
}

}  // extern "C"
