// extern "C" entry points of libdpb.so — see include/dpb.h for the contract
// and the reference interface each one replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/dpb.h"
#include "dpb_internal.h"
#include "dpb_launch.h"

namespace dpb {
int op_batch_statistics(const float*, int64_t, int64_t, int64_t, int64_t, float*, float*,
                        cudaStream_t);
int op_batchnorm_apply(const float*, int64_t, int64_t, int64_t, int64_t, const float*,
                       const float*, const float*, const float*, int, float*, cudaStream_t);
int op_batchnorm_backward(const float*, const float*, int64_t, int64_t, int64_t, int64_t,
                          const float*, const float*, const float*, float*, float*, float*,
                          cudaStream_t);
int op_conv2d_forward(const float*, int64_t, int64_t, int64_t, int64_t, const float*, int64_t,
                      int, int, float*, cudaStream_t);
int op_conv2d_backward(const float*, const float*, int64_t, int64_t, int64_t, int64_t,
                       const float*, int64_t, int, int, float*, float*, cudaStream_t);
int op_relu_forward(const float*, int64_t, float*, cudaStream_t);
int op_relu_backward(const float*, const float*, int64_t, float*, cudaStream_t);
int op_concat(int, const float* const*, const int64_t*, int64_t, int64_t, float*, int64_t, int, cudaStream_t);
}  // namespace dpb

using dpb::Block;
using dpb::fail;

static Block* B(dpb_block* p) { return reinterpret_cast<Block*>(p); }

static int op_status(int e, const char* what) {
  if (e == 0) return DPB_OK;
  return dpb::cuda_fail(static_cast<cudaError_t>(e), what);
}

static int check_nhw(int64_t n, int64_t c, int64_t h, int64_t w) {
  if (n < 1 || c < 1 || h < 1 || w < 1) return fail(DPB_SHAPE_ERROR, "invalid shape");
  return DPB_OK;
}

// --- host-side model arithmetic ------------------------------------------------
// Restated from densenet.hpp:141-180 (net_geometry), :234-275
// (count_parameters) and peak_model.hpp:37-158 (predict_peak_elements),
// pre-activation only (every configuration of BASELINE.json).
namespace {

struct Cfg {
  std::vector<int> blocks;
  int64_t k = 12;
  bool bottleneck = true;
  double compression = 1.0;
  int64_t classes = 10;
  int64_t c0 = 24;
};

int make_cfg(int nblocks, const int32_t* blocks, int32_t k, int32_t bottleneck,
             double compression, int32_t classes, int32_t c0, Cfg* out) {
  if (nblocks < 1 || blocks == nullptr) return fail(DPB_CONFIG_ERROR, "no dense blocks configured");
  for (int i = 0; i < nblocks; ++i)
    if (blocks[i] < 1) return fail(DPB_CONFIG_ERROR, "block size must be >= 1");
  if (k < 1) return fail(DPB_CONFIG_ERROR, "growth rate must be >= 1");
  if (!(compression > 0.0) || compression > 1.0)
    return fail(DPB_CONFIG_ERROR, "compression must be in (0, 1]");
  if (classes < 1) return fail(DPB_CONFIG_ERROR, "num_classes must be >= 1");
  out->blocks.assign(blocks, blocks + nblocks);
  out->k = k;
  out->bottleneck = bottleneck != 0;
  out->compression = compression;
  out->classes = classes;
  out->c0 = c0 > 0 ? c0 : 2 * k;  // build_config default, densenet.hpp:83
  return DPB_OK;
}

int64_t trans_out(const Cfg& c, int64_t ch) {
  return static_cast<int64_t>(std::floor(c.compression * static_cast<double>(ch)));
}

}  // namespace

extern "C" {

const char* dpb_last_error(void) { return dpb::g_last_error.c_str(); }
const char* dpb_version(void) { return "dpb 0.1 sm_100a"; }

int dpb_block_plan(const dpb_block_desc* desc, dpb_arena_sizes* out) {
  const int rc = dpb::validate(desc);
  if (rc) return rc;
  if (!out) return fail(DPB_CONFIG_ERROR, "null output");
  dpb::plan_arena(*desc, out);
  return DPB_OK;
}

int dpb_block_param_elems(const dpb_block_desc* desc, int64_t* pe, int64_t* se) {
  dpb_arena_sizes s;
  const int rc = dpb_block_plan(desc, &s);
  if (rc) return rc;
  if (pe) *pe = s.param_elems;
  if (se) *se = s.stat_elems;
  return DPB_OK;
}

int dpb_block_create(const dpb_block_desc* desc, int device, void* stream, dpb_block** out) {
  Block* b = nullptr;
  dpb::DeviceGuard dg(device);
  const int rc = dpb::create(desc, device, stream, &b);
  if (rc) return rc;
  *out = reinterpret_cast<dpb_block*>(b);
  return DPB_OK;
}

int dpb_block_destroy(dpb_block* blk) {
  if (!blk) return DPB_OK;
  dpb::DeviceGuard dg(B(blk)->device);
  dpb::destroy(B(blk));
  return DPB_OK;
}

int dpb_block_set_stream(dpb_block* blk, void* stream) {
  if (!blk) return fail(DPB_CONFIG_ERROR, "null block");
  B(blk)->stream = static_cast<cudaStream_t>(stream);
  return DPB_OK;
}

int dpb_block_arena(dpb_block* blk, dpb_arena_sizes* out, void** base) {
  if (!blk) return fail(DPB_CONFIG_ERROR, "null block");
  if (out) *out = B(blk)->sz;
  if (base) *base = B(blk)->arena;
  return DPB_OK;
}

int dpb_block_forward(dpb_block* blk, const float* x_in, const float* params, float* running,
                      int update_running) {
  if (!blk || !x_in || !params) return fail(DPB_CONFIG_ERROR, "null argument");
  if (update_running && !running) return fail(DPB_CONFIG_ERROR, "running stats required");
  dpb::DeviceGuard dg(B(blk)->device);
  return dpb::block_forward(B(blk), x_in, params, running, update_running, 0);
}

int dpb_block_forward_eval(dpb_block* blk, const float* x_in, const float* params,
                           const float* running) {
  if (!blk || !x_in || !params || !running) return fail(DPB_CONFIG_ERROR, "null argument");
  dpb::DeviceGuard dg(B(blk)->device);
  return dpb::block_forward(B(blk), x_in, params, const_cast<float*>(running), 0, 1);
}

int dpb_block_backward(dpb_block* blk, const float* params, float* grad_acc, float* grads) {
  if (!blk || !params || !grad_acc || !grads) return fail(DPB_CONFIG_ERROR, "null argument");
  dpb::DeviceGuard dg(B(blk)->device);
  return dpb::block_backward(B(blk), params, grad_acc, grads);
}

int dpb_block_read_feats(dpb_block* blk, float* dst) {
  if (!blk || !dst) return fail(DPB_CONFIG_ERROR, "null argument");
  dpb::DeviceGuard dg(B(blk)->device);
  return dpb::read_feats(B(blk), dst);
}
int dpb_block_read_z(dpb_block* blk, float* dst) {
  if (!blk || !dst) return fail(DPB_CONFIG_ERROR, "null argument");
  dpb::DeviceGuard dg(B(blk)->device);
  return dpb::read_z(B(blk), dst);
}
int dpb_block_read_stats(dpb_block* blk, float* dst) {
  if (!blk || !dst) return fail(DPB_CONFIG_ERROR, "null argument");
  dpb::DeviceGuard dg(B(blk)->device);
  return dpb::read_stats(B(blk), dst);
}

int dpb_sync(dpb_block* blk) {
  if (!blk) return fail(DPB_CONFIG_ERROR, "null block");
  dpb::DeviceGuard dg(B(blk)->device);
  const cudaError_t e = cudaStreamSynchronize(B(blk)->stream);
  if (e != cudaSuccess) return dpb::cuda_fail(e, "stream synchronize");
  return DPB_OK;
}

int64_t dpb_block_launch_count(dpb_block* blk) { return blk ? B(blk)->launches : -1; }

int dpb_block_trace(dpb_block* blk, int32_t* counts, int max_nodes, double* flops, int* nodes) {
  if (!blk || !nodes) return fail(DPB_CONFIG_ERROR, "null argument");
  const dpb::BlockTrace& t = B(blk)->trace;
  const int n = static_cast<int>(t.counts.size() / 3);
  *nodes = n;
  if (counts)
    for (int i = 0; i < 3 * n && i < 3 * max_nodes; ++i) counts[i] = t.counts[static_cast<size_t>(i)];
  if (flops)
    for (int w = 0; w < 3; ++w)
      for (int k = 0; k < dpb::BlockTrace::kKinds; ++k) flops[w * dpb::BlockTrace::kKinds + k] = t.flops[w][k];
  return DPB_OK;
}

int dpb_block_memory_stats(dpb_block* blk, dpb_memory_stats* out) {
  if (!blk || !out) return fail(DPB_CONFIG_ERROR, "null argument");
  B(blk)->tracker->snapshot(out);
  return DPB_OK;
}

int dpb_block_profile(dpb_block* blk, int enable) {
  if (!blk) return fail(DPB_CONFIG_ERROR, "null block");
  dpb::profile_enable(B(blk), enable);
  return DPB_OK;
}

int dpb_block_profile_read(dpb_block* blk, dpb_kernel_stat* out, int max, int* count) {
  if (!blk || !out || !count) return fail(DPB_CONFIG_ERROR, "null argument");
  dpb::DeviceGuard dg(B(blk)->device);
  return dpb::profile_read(B(blk), out, max, count);
}

// Efficient: the planned arena (features + bottleneck outputs + stats +
// gradient slots + scratch).  Naive store-everything (Naive strategy of
// graph.hpp:279-310 for one block, fp32 like the reference): every layer's
// concat, BN_a/ReLU output, z, BN_b/ReLU output and y retained, plus every
// backward buffer (4 transients per layer) and the accumulator.
int dpb_block_memory(const dpb_block_desc* desc, int64_t* eff, int64_t* naive) {
  dpb_arena_sizes s;
  const int rc = dpb_block_plan(desc, &s);
  if (rc) return rc;
  if (eff) *eff = s.total_bytes;
  if (naive) {
    const int64_t M = desc->n * desc->h * desc->w;
    int64_t e = M * desc->c0;  // block input
    for (int l = 0; l < desc->m; ++l) {
      const int64_t c = desc->c0 + static_cast<int64_t>(l) * desc->k;
      e += 2 * c * M;                 // cat, act_a
      e += 2LL * desc->bk * M;        // z, act_b
      e += static_cast<int64_t>(desc->k) * M;  // y
      e += (2LL * desc->bk + 2 * c) * M;       // t0..t3
    }
    const int64_t C = desc->c0 + static_cast<int64_t>(desc->m) * desc->k;
    e += 2 * C * M;  // block-output concat + accumulator
    const int64_t S = desc->dtype == DPB_BF16 ? 2 : 4;
    *naive = e * S;
  }
  return DPB_OK;
}

// --- per-op entry points ---------------------------------------------------------
int dpb_op_batch_statistics(const float* x, int64_t n, int64_t c, int64_t h, int64_t w,
                            float* mean, float* var, void* stream) {
  if (int rc = check_nhw(n, c, h, w)) return rc;
  return op_status(dpb::op_batch_statistics(x, n, c, h, w, mean, var,
                                            static_cast<cudaStream_t>(stream)),
                   "batch_statistics");
}
int dpb_op_batchnorm_apply(const float* x, int64_t n, int64_t c, int64_t h, int64_t w,
                           const float* gamma, const float* beta, const float* mean,
                           const float* var, int relu, float* dst, void* stream) {
  if (int rc = check_nhw(n, c, h, w)) return rc;
  return op_status(dpb::op_batchnorm_apply(x, n, c, h, w, gamma, beta, mean, var, relu, dst,
                                           static_cast<cudaStream_t>(stream)),
                   "batchnorm_apply");
}
int dpb_op_batchnorm_backward(const float* gy, const float* x, int64_t n, int64_t c, int64_t h,
                              int64_t w, const float* gamma, const float* mean, const float* var,
                              float* gx, float* dg, float* db, void* stream) {
  if (int rc = check_nhw(n, c, h, w)) return rc;
  return op_status(dpb::op_batchnorm_backward(gy, x, n, c, h, w, gamma, mean, var, gx, dg, db,
                                              static_cast<cudaStream_t>(stream)),
                   "batchnorm_backward");
}
int dpb_op_conv2d_forward(const float* x, int64_t n, int64_t cin, int64_t h, int64_t w,
                          const float* wt, int64_t cout, int64_t kernel, int64_t pad,
                          float* dst, void* stream) {
  if (int rc = check_nhw(n, cin, h, w)) return rc;
  if (cout < 1 || kernel < 1 || pad < 0) return fail(DPB_SHAPE_ERROR, "invalid conv params");
  if (h + 2 * pad - kernel + 1 < 1 || w + 2 * pad - kernel + 1 < 1)
    return fail(DPB_SHAPE_ERROR, "conv output collapses to zero size");  // ops.hpp:305-308
  return op_status(dpb::op_conv2d_forward(x, n, cin, h, w, wt, cout, static_cast<int>(kernel),
                                          static_cast<int>(pad),
                                          dst, static_cast<cudaStream_t>(stream)),
                   "conv2d_forward");
}
int dpb_op_conv2d_backward(const float* gy, const float* x, int64_t n, int64_t cin, int64_t h,
                           int64_t w, const float* wt, int64_t cout, int64_t kernel, int64_t pad,
                           float* gx, float* gw, void* stream) {
  if (int rc = check_nhw(n, cin, h, w)) return rc;
  if (cout < 1 || kernel < 1 || pad < 0) return fail(DPB_SHAPE_ERROR, "invalid conv params");
  if (h + 2 * pad - kernel + 1 < 1 || w + 2 * pad - kernel + 1 < 1)
    return fail(DPB_SHAPE_ERROR, "conv output collapses to zero size");
  return op_status(dpb::op_conv2d_backward(gy, x, n, cin, h, w, wt, cout,
                                           static_cast<int>(kernel), static_cast<int>(pad), gx,
                                           gw, static_cast<cudaStream_t>(stream)),
                   "conv2d_backward");
}

static int concat_check(int count, const void* parts, const int64_t* channels, int64_t n, int64_t h, int64_t w,
                        int64_t whole_c) {
  if (count < 1 || !parts || !channels) return fail(DPB_SHAPE_ERROR, "concat of zero inputs");  // ops.hpp:55
  if (int rc = check_nhw(n, whole_c, h, w)) return rc;
  int64_t total = 0;
  for (int i = 0; i < count; ++i) {
    if (channels[i] < 1) return fail(DPB_SHAPE_ERROR, "concat input with no channels");
    total += channels[i];
  }
  if (total != whole_c)  // ops.hpp:66-69 (forward) / :94-98 (backward)
    return fail(DPB_CAPACITY_ERROR, "concat channel sum " + std::to_string(total) + " != dst channels " +
                                        std::to_string(whole_c));
  return DPB_OK;
}

int dpb_op_concat_forward(int count, const float* const* inputs, const int64_t* channels, int64_t n, int64_t h,
                          int64_t w, float* dst, int64_t dst_c, void* stream) {
  if (int rc = concat_check(count, inputs, channels, n, h, w, dst_c)) return rc;
  return op_status(dpb::op_concat(count, inputs, channels, n, h * w, dst, dst_c, 0,
                                  static_cast<cudaStream_t>(stream)),
                   "concat_forward");
}
int dpb_op_concat_backward(const float* grad_out, int64_t n, int64_t c, int64_t h, int64_t w, int count,
                           const int64_t* channels, float* const* grads, void* stream) {
  if (int rc = concat_check(count, grads, channels, n, h, w, c)) {
    if (rc == DPB_CAPACITY_ERROR) return fail(DPB_SHAPE_ERROR, dpb::g_last_error);  // ops.hpp:94-98: ShapeError
    return rc;
  }
  return op_status(dpb::op_concat(count, grads, channels, n, h * w, const_cast<float*>(grad_out), c, 1,
                                  static_cast<cudaStream_t>(stream)),
                   "concat_backward");
}
int dpb_op_relu_forward(const float* x, int64_t count, float* dst, void* stream) {
  if (count < 0) return fail(DPB_SHAPE_ERROR, "negative element count");
  return op_status(dpb::op_relu_forward(x, count, dst, static_cast<cudaStream_t>(stream)), "relu_forward");
}
int dpb_op_relu_backward(const float* grad_y, const float* ref, int64_t count, float* grad_x, void* stream) {
  if (count < 0) return fail(DPB_SHAPE_ERROR, "negative element count");
  return op_status(dpb::op_relu_backward(grad_y, ref, count, grad_x, static_cast<cudaStream_t>(stream)),
                   "relu_backward");
}

// --- host-side model arithmetic ----------------------------------------------------
int dpb_count_parameters(int nblocks, const int32_t* blocks, int32_t k, int32_t bottleneck,
                         double compression, int32_t classes, int32_t c0, int32_t in_c,
                         int64_t* out) {
  Cfg cfg;
  if (int rc = make_cfg(nblocks, blocks, k, bottleneck, compression, classes, c0, &cfg)) return rc;
  const int64_t bk = 4 * cfg.k;
  int64_t total = static_cast<int64_t>(in_c) * cfg.c0 * 9;  // stem 3x3
  int64_t c = cfg.c0;
  for (size_t b = 0; b < cfg.blocks.size(); ++b) {
    for (int l = 0; l < cfg.blocks[b]; ++l) {
      total += 2 * c;
      if (cfg.bottleneck) total += c * bk + 2 * bk + bk * cfg.k * 9;
      else total += c * cfg.k * 9;
      c += cfg.k;
    }
    if (b + 1 < cfg.blocks.size()) {
      const int64_t t = trans_out(cfg, c);
      total += 2 * c + c * t;
      c = t;
    }
  }
  total += 2 * c + c * cfg.classes + cfg.classes;
  *out = total;
  return DPB_OK;
}

int dpb_predict_peak_elements(int nblocks, const int32_t* blocks, int32_t k, int32_t bottleneck,
                              double compression, int32_t classes, int32_t c0, int32_t strategy,
                              int64_t batch, int32_t in_c, int32_t in_h, int32_t in_w,
                              int64_t* out) {
  Cfg cfg;
  if (int rc = make_cfg(nblocks, blocks, k, bottleneck, compression, classes, c0, &cfg)) return rc;
  if (batch < 1) return fail(DPB_CONFIG_ERROR, "batch must be >= 1");
  if (in_c < 1 || in_h < 1 || in_w < 1) return fail(DPB_CONFIG_ERROR, "invalid input shape");
  if (strategy < 0 || strategy > 2) return fail(DPB_CONFIG_ERROR, "unknown strategy");
  const int64_t N = batch, K = cfg.k, bk = 4 * cfg.k;
  int64_t owned = cfg.c0 * static_cast<int64_t>(in_h) * in_w * N;
  std::vector<int64_t> cat, bnpool, bnunit, gtr, accs;
  int64_t c = cfg.c0, h = in_h, w = in_w;
  const size_t nb = cfg.blocks.size();
  for (size_t b = 0; b < nb; ++b) {
    const int64_t hw = h * w;
    for (int l = 0; l < cfg.blocks[b]; ++l) {
      const int64_t cl = c + l * K;
      cat.push_back(cl * hw * N);
      bnpool.push_back(cl * hw * N);
      if (cfg.bottleneck) {
        bnpool.push_back(bk * hw * N);
        bnunit.push_back((cl + bk) * hw * N);
        owned += bk * hw * N + K * hw * N;
        gtr.insert(gtr.end(), {bk * hw * N, bk * hw * N, cl * hw * N, cl * hw * N});
      } else {
        bnunit.push_back(cl * hw * N);
        owned += K * hw * N;
        gtr.insert(gtr.end(), {cl * hw * N, cl * hw * N});
      }
    }
    const int64_t cout = c + cfg.blocks[b] * K;
    cat.push_back(cout * hw * N);
    accs.push_back(cout * hw * N);
    if (b + 1 < nb) {
      if (h < 2 || w < 2) return fail(DPB_CONFIG_ERROR, "spatial size collapses");
      const int64_t t = trans_out(cfg, cout);
      if (t < 1) return fail(DPB_CONFIG_ERROR, "compression collapses channels to 0");
      const int64_t hh = (h - 2) / 2 + 1, ww = (w - 2) / 2 + 1;
      bnpool.push_back(cout * hw * N);
      bnunit.push_back(cout * hw * N);
      owned += t * hw * N + t * hh * ww * N;
      gtr.insert(gtr.end(), {t * hw * N, cout * hw * N});
      c = t;
      h = hh;
      w = ww;
    } else {
      bnpool.push_back(cout * hw * N);
      bnunit.push_back(cout * hw * N);
      owned += cout * N + cfg.classes * N;
      gtr.insert(gtr.end(), {cout * N, cout * hw * N});
    }
  }
  auto sum = [](const std::vector<int64_t>& v) {
    int64_t t = 0;
    for (int64_t x : v) t += x;
    return t;
  };
  auto mx = [](const std::vector<int64_t>& v) {
    int64_t t = 0;
    for (int64_t x : v) t = std::max(t, x);
    return t;
  };
  const int64_t region = std::max(mx(gtr), mx(accs));
  int64_t params = 0;
  if (int rc = dpb_count_parameters(nblocks, blocks, k, bottleneck, compression, classes, c0, in_c,
                                    &params))
    return rc;
  for (int i = 0; i < 6; ++i) out[i] = 0;
  out[DPB_ARENA_PARAMS] = 2 * params;
  out[DPB_ARENA_SCRATCH] = cfg.classes * N;
  if (strategy == 0) {
    out[DPB_ARENA_FEATURE_OWNED] = owned + sum(cat) + sum(bnpool) + sum(gtr) + sum(accs);
  } else if (strategy == 1) {
    out[DPB_ARENA_FEATURE_OWNED] = owned + sum(cat) + sum(bnpool);
    out[DPB_ARENA_SHARED_GRAD] = 4 * region;
  } else {
    out[DPB_ARENA_FEATURE_OWNED] = owned;
    out[DPB_ARENA_SHARED1] = mx(cat);
    out[DPB_ARENA_SHARED2] = mx(bnunit);
    out[DPB_ARENA_SHARED_GRAD] = 4 * region;
  }
  return DPB_OK;
}

// Rng::normal (rng.hpp:36-49) over std::mt19937_64, whose bit stream the C++
// standard fixes, so parameter init and synthetic inputs are reproducible.
int dpb_rng_fill_normal(uint64_t seed, float* dst, int64_t count) {
  if (!dst || count < 0) return fail(DPB_CONFIG_ERROR, "bad rng arguments");
  std::mt19937_64 eng(seed);
  bool have = false;
  double spare = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    double v;
    if (have) {
      have = false;
      v = spare;
    } else {
      double u1 = static_cast<double>(eng() >> 11) * 0x1.0p-53;
      const double u2 = static_cast<double>(eng() >> 11) * 0x1.0p-53;
      while (u1 <= 0.0) u1 = static_cast<double>(eng() >> 11) * 0x1.0p-53;
      const double r = std::sqrt(-2.0 * std::log(u1));
      const double th = 2.0 * 3.14159265358979323846 * u2;
      spare = r * std::sin(th);
      have = true;
      v = r * std::cos(th);
    }
    dst[i] = static_cast<float>(v);
  }
  return DPB_OK;
}

}  // extern "C"
