// Block plan, HBM arena and the forward/backward orchestration behind the
// C ABI (include/dpb.h).
//
// Reference mapping (paths under /root/reference/proj/include/denseplan):
//   plan_arena()        PoolRegion/GradPool/BufferPool sizing, graph.hpp:28-127,
//                       :456-482, :602-609 — but Shared1/Shared2 are 0 here
//   block_forward()     GraphPlan::forward layer loop, graph.hpp:747-760,
//                       forward_layer :618-670
//   block_backward()    backward_block :1054-1063 -> backward_layer :856-945
//                       with rematerialize :831-854 folded into the kernels
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <new>
#include <string>

#include "../../include/dpb.h"
#include "dpb_common.cuh"
#include "dpb_kernels.cuh"
#include "dpb_simt.cuh"
#include "dpb_internal.h"
#include "dpb_launch.h"

namespace dpb {

thread_local std::string g_last_error;

const char* const kKernelCatNames[KC_COUNT] = {
    "pack", "channel_stats", "finalize", "conv1x1_fwd", "conv3x3_fwd", "conv3x3_dgrad",
    "conv3x3_wgrad", "conv1x1_dgrad", "conv1x1_wgrad", "reduce_wgrad", "bn_apply_accumulate",
    "running_update"};

static cudaEvent_t next_event(Block* b) {
  if (b->ev_used == b->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    b->ev_pool.push_back(e);
  }
  return b->ev_pool[b->ev_used++];
}

LaunchScope::LaunchScope(Block* blk, int cat_, double bytes, double flops, double bytes_8d)
    : b(blk), cat(cat_) {
  b->launches++;
  current_cat() = cat_;
  if (!b->prof) return;
  ProfRec r{cat_, next_event(b), next_event(b), bytes, flops, bytes_8d};
  cudaEventRecord(r.start, b->stream);
  idx = static_cast<int>(b->recs.size());
  b->recs.push_back(r);
}

LaunchScope::~LaunchScope() {
  current_cat() = -1;
  if (idx >= 0) cudaEventRecord(b->recs[idx].stop, b->stream);
  // debugging aid: DPB_DEBUG_SYNC=1 synchronizes after every launch and names
  // the first launch that faults (category, launch ordinal)
  static const bool dbg = std::getenv("DPB_DEBUG_SYNC") != nullptr;
  if (dbg) {
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess)
      std::fprintf(stderr, "[dpb] launch %lld (category %d) failed: %s\n",
                   static_cast<long long>(b->launches), cat, cudaGetErrorString(e));
  }
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(DPB_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

static int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

int validate(const dpb_block_desc* d) {
  if (d == nullptr) return fail(DPB_CONFIG_ERROR, "null descriptor");
  if (d->n < 1 || d->h < 1 || d->w < 1 || d->c0 < 1 || d->m < 1 || d->k < 1 || d->bk < 1)
    return fail(DPB_SHAPE_ERROR, "invalid block shape (every extent must be >= 1)");
  if (d->dtype != DPB_FP32 && d->dtype != DPB_BF16)
    return fail(DPB_CONFIG_ERROR, "dtype must be DPB_FP32 or DPB_BF16");
  if (d->layout != DPB_NCHW && d->layout != DPB_NHWC)
    return fail(DPB_CONFIG_ERROR, "layout must be DPB_NCHW or DPB_NHWC");
  // Shape4::elems overflow guard (tensor.hpp:26-39): int64_max / 16
  const unsigned __int128 lim = static_cast<unsigned __int128>(INT64_MAX / 16);
  const int64_t C = static_cast<int64_t>(d->c0) + static_cast<int64_t>(d->m) * d->k;
  unsigned __int128 p = static_cast<unsigned __int128>(d->n) * d->h;
  p *= d->w;
  if (p > lim) return fail(DPB_SIZE_OVERFLOW_ERROR, "pixel count overflows");
  if (p * static_cast<unsigned __int128>(C) > lim ||
      p * static_cast<unsigned __int128>(d->bk) * d->m > lim)
    return fail(DPB_SIZE_OVERFLOW_ERROR, "block tensor overflows element count");
  if (C > (1 << 20) || d->bk > (1 << 16))
    return fail(DPB_CONFIG_ERROR, "channel count beyond supported range");
  return DPB_OK;
}

Geometry geometry(const dpb_block_desc& d) {
  Geometry g;
  g.M = d.n * d.h * d.w;
  g.C = d.c0 + d.m * d.k;
  g.Cp = (g.C + 3) / 4 * 4;
  g.cmax = d.c0 + (d.m - 1) * d.k;
  g.cmaxp = (g.cmax + 3) / 4 * 4;
  g.P = static_cast<int>((g.M + 127) / 128);
  g.Pmax = g.P;
  if (d.dtype == DPB_BF16 && tc_supported(d))
    g.Pmax = static_cast<int>(std::max<int64_t>(g.P, tc_halo_partials(d)));
  g.S = 4;  // features and bottleneck outputs are stored fp32
  return g;
}

// Split-K choice for the weight-gradient GEMMs (K = pixels): aim for ~2 waves
// of 148 SMs, at least 256 pixels per split.
int64_t wgrad_chunk(int64_t M, int64_t tiles) {
  int64_t splits = std::max<int64_t>(1, 296 / std::max<int64_t>(1, tiles));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, M / 256));
  int64_t chunk = (M + splits - 1) / splits;
  chunk = align_up(chunk, kBK);
  return chunk;
}

static int bn_tile(int64_t n) {
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 48) return 48;
  return 64;
}

// Pre-tiled bf16 weight images of the tensor-core path: W1 (1x1 forward) per
// layer, then W2 (halo forward) and W2^T (halo dgrad) per layer.
static int64_t weight_image_bytes(const dpb_block_desc& d) {
  int64_t w1 = 0, w1b = 0;
  for (int l = 0; l < d.m; ++l) {
    w1 += tc2_w1_tile_bytes(d, l);
    w1b += tc2_w1b_layer_bytes(d, l);
  }
  const HaloPlan hp = tc_halo_plan(d);
  return align_up(w1, 256) + align_up(hp.fwd_layer_bytes * d.m, 256) +
         align_up(hp.bwd_layer_bytes * d.m, 256) + align_up(w1b, 256);
}

// Partials of the split-K 1x1 forward (tensor-core path): the widest layer's
// ks x M x bk fp32.
static int64_t zsplit_bytes(const dpb_block_desc& d) {
  if (d.dtype != DPB_BF16 || !tc_supported(d)) return 0;
  const int64_t M = d.n * d.h * d.w;
  int64_t most = 0;
  for (int l = 0; l < d.m; ++l) {
    for (int ns = 1; ns <= 2; ++ns) {  // the column split the stage width may need
      const int ks = tc2_fwd_ksplit(M, d.c0 + l * d.k, 148, ns);
      if (ks > 1) most = std::max<int64_t>(most, ks * M * d.bk * 4);
    }
  }
  return most;
}

void plan_arena(const dpb_block_desc& d, dpb_arena_sizes* s) {
  const Geometry g = geometry(d);
  std::memset(s, 0, sizeof(*s));
  int64_t off = 0;
  auto take = [&](int64_t bytes, int64_t* o, int64_t* b) {
    *o = off;
    *b = bytes;
    off = align_up(off + bytes, 256);
  };
  take(g.M * g.Cp * g.S, &s->feat_offset, &s->feat_bytes);
  take(static_cast<int64_t>(d.m) * g.M * d.bk * g.S, &s->z_offset, &s->z_bytes);
  take((2 * g.Cp + 2LL * d.m * d.bk) * 4, &s->stats_offset, &s->stats_bytes);
  take(d.layout == DPB_NCHW ? g.M * g.Cp * 4 : 0, &s->acc_offset, &s->acc_bytes);
  take(2 * g.M * d.bk * 4, &s->g0_offset, &s->g0_bytes);
  // g1 double-buffered by layer parity: the tail of layer l's accumulate
  // overlaps layer l-1's dgrads (split_apply)
  take(2 * g.M * g.cmaxp * 4, &s->g1_offset, &s->g1_bytes);
  // scratch: partials | wgrad partials | BN-backward coefficients
  int64_t wmax = 0;
  for (int l = 0; l < d.m; ++l) {
    const int64_t c = d.c0 + static_cast<int64_t>(l) * d.k;
    {
      const int64_t rows = 9LL * d.bk, cols = d.k;
      const int bn = bn_tile(cols);
      const int64_t tiles = ((rows + 127) / 128) * ((cols + bn - 1) / bn);
      const int64_t chunk = wgrad_chunk(g.M, tiles);
      const int64_t splits = (g.M + chunk - 1) / chunk;
      wmax = std::max(wmax, splits * rows * cols);
    }
    {
      const int64_t rows = d.bk, cols = c;
      const int64_t tiles = ((rows + 63) / 64) * ((cols + 63) / 64);
      const int64_t chunk = wgrad_chunk(g.M, tiles);
      const int64_t splits = (g.M + chunk - 1) / chunk;
      wmax = std::max(wmax, splits * rows * cols);
    }
    if (d.dtype == DPB_BF16 && tc_supported(d)) {
      wmax = std::max<int64_t>(wmax, tc_halo_wgrad_splits(d) * 9LL * d.bk * d.k);
      const int64_t c3 = tc_wgrad_chunk(g.M, (9LL * d.bk + 127) / 128);
      wmax = std::max<int64_t>(wmax, ((g.M + c3 - 1) / c3) * 9LL * d.bk * d.k);
      const int64_t c1 = tc_wgrad_chunk(g.M, (c + 127) / 128);
      wmax = std::max<int64_t>(wmax, ((g.M + c1 - 1) / c1) * c * d.bk);
      wmax = std::max<int64_t>(wmax, tc2_wgrad_wpart_elems(d, l));
    }
  }
  const int64_t pbytes = std::max<int64_t>(static_cast<int64_t>(g.Pmax) * std::max<int64_t>(g.C, d.bk) * 16,
                                          zsplit_bytes(d) > 0 ? (g.M + 31) / 32 * d.bk * 16 : 0);
  const int64_t scratch = align_up(pbytes, 256) + align_up(wmax * 4, 256) +
                          align_up((4LL * d.bk + 4 * g.cmaxp) * 4, 256) + align_up(zsplit_bytes(d), 256);
  take(scratch, &s->scratch_offset, &s->scratch_bytes);
  // pre-tiled bf16 weight operands of the tensor-core path (counted as scratch)
  if (d.dtype == DPB_BF16 && tc_supported(d)) {
    const int64_t wt = weight_image_bytes(d);
    s->scratch_bytes += wt;
    off = align_up(off + wt, 256);
  }
  s->total_bytes = off;
  s->shared1_bytes = 0;
  s->shared2_bytes = 0;
  int64_t pe = 0, se = 0;
  for (int l = 0; l < d.m; ++l) {
    const int64_t c = d.c0 + static_cast<int64_t>(l) * d.k;
    pe += 2 * c + d.bk * c + 2LL * d.bk + 9LL * d.k * d.bk;
    se += 2 * c + 2LL * d.bk;
  }
  s->param_elems = pe;
  s->stat_elems = se;
}

// --- launch helpers -----------------------------------------------------------

template <int BM, int BN, class Op>
static void launch_gemm(Block* b, const Op& op, dim3 grid, size_t dyn) {
  launch(gemm_kernel<BM, BN, Op>, grid, kThreads, dyn, b->stream, op);
}

// Dispatch on the N tile for ops whose N is a runtime channel count.
template <int BM, template <typename> class OpT, typename S>
static void gemm_bn(Block* b, const LayerArgs<S>& a, int64_t rows, int64_t cols, int gz) {
  OpT<S> op{a};
  const size_t dyn = OpT<S>::smem(a);
  const int bn = bn_tile(cols);
  const dim3 grid(static_cast<unsigned>((rows + BM - 1) / BM),
                  static_cast<unsigned>((cols + bn - 1) / bn), gz);
  switch (bn) {
    case 16: launch_gemm<BM, 16>(b, op, grid, dyn); break;
    case 32: launch_gemm<BM, 32>(b, op, grid, dyn); break;
    case 48: launch_gemm<BM, 48>(b, op, grid, dyn); break;
    default: launch_gemm<BM, 64>(b, op, grid, dyn); break;
  }
}

template <int BM, template <typename, int> class OpT, typename S>
static void gemm_bn2(Block* b, const LayerArgs<S>& a, int64_t rows, int64_t cols, int gz) {
  const int bn = bn_tile(cols);
  const unsigned gx = static_cast<unsigned>((rows + BM - 1) / BM);
  const unsigned gy = static_cast<unsigned>((cols + bn - 1) / bn);
  switch (bn) {
    case 16: launch_gemm<BM, 16>(b, OpT<S, 16>{a}, dim3(gx, gy, gz), OpT<S, 16>::smem(a)); break;
    case 32: launch_gemm<BM, 32>(b, OpT<S, 32>{a}, dim3(gx, gy, gz), OpT<S, 32>::smem(a)); break;
    case 48: launch_gemm<BM, 48>(b, OpT<S, 48>{a}, dim3(gx, gy, gz), OpT<S, 48>::smem(a)); break;
    default: launch_gemm<BM, 64>(b, OpT<S, 64>{a}, dim3(gx, gy, gz), OpT<S, 64>::smem(a)); break;
  }
}

static unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

template <typename S>
static LayerArgs<S> layer_args(Block* b, const float* params, int l) {
  const dpb_block_desc& d = b->d;
  const Geometry& g = b->g;
  LayerArgs<S> a{};
  a.M = g.M;
  a.H = static_cast<int>(d.h);
  a.W = static_cast<int>(d.w);
  a.C = static_cast<int>(g.Cp);
  a.Ca = static_cast<int>(b->acc_pitch > 0 ? b->acc_pitch : g.Cp);
  a.c = d.c0 + l * d.k;
  a.cg = (a.c + 3) / 4 * 4;
  a.bk = d.bk;
  a.k = d.k;
  a.feat = static_cast<S*>(b->feat);
  a.z = static_cast<S*>(b->z) + static_cast<int64_t>(l) * g.M * d.bk;
  const float* p = params + b->param_off[l];
  a.gamma_a = p;
  a.beta_a = p + a.c;
  a.w1 = p + 2 * a.c;
  a.gamma_b = a.w1 + static_cast<int64_t>(d.bk) * a.c;
  a.beta_b = a.gamma_b + d.bk;
  a.w2 = a.beta_b + d.bk;
  a.amean = b->fstat;
  a.avar = b->fstat + g.Cp;
  a.bmean = b->zstat + static_cast<int64_t>(l) * 2 * d.bk;
  a.bvar = a.bmean + d.bk;
  a.acc = b->acc_cur;
  a.g0 = b->g0;
  a.g1 = b->g1 + (l & 1) * g.M * g.cmaxp;  // parity buffer
  a.bnb_bwd = b->bnb_bwd;
  a.part = b->part;
  a.wpart = b->wpart;
  return a;
}

template <typename S>
static void forward_impl(Block* b, const float* x_in, const float* params, float* running,
                         int update_running, int eval) {
  const dpb_block_desc& d = b->d;
  const Geometry& g = b->g;
  S* feat = static_cast<S*>(b->feat);
  const int64_t hw = d.h * d.w;
  const double M = static_cast<double>(g.M), Sb = g.S;
  // block input -> channels [0, c0) of the feature buffer (zero-copy concat);
  // the whole-network step writes it there directly (x_in == feat, NHWC)
  if (static_cast<const void*>(x_in) != b->feat || d.layout != DPB_NHWC) {
    LaunchScope ls(b, KC_PACK, M * d.c0 * (4 + Sb), 0, M * d.c0 * (4 + 2.0));
    if (d.layout == DPB_NCHW) {
      dim3 grid(blocks_for(hw, 32), blocks_for(d.c0, 32), static_cast<unsigned>(d.n));
      launch(k_nchw_to_nhwc<S>, grid, dim3(32, 8), 0, b->stream, x_in, d.n, d.c0, hw, feat,
                                                             static_cast<int>(g.Cp), 0);
    } else {
      launch(k_nhwc_copy<S>, blocks_for(g.M * d.c0, 256), 256, 0, b->stream, 
          x_in, d.c0, g.M, d.c0, feat, static_cast<int>(g.Cp), 0);
    }
  }
  if (b->tc) {
    LaunchScope ls(b, KC_PACK, 0, 0, 0);
    b->launches--;  // counted inside tc2_pretile_w1
    tc2_pretile_w1(b, params);
    tc_pretile_w2(b, params, true);
  }
  const double count = M;
  float* fmean = b->fstat;
  float* fvar = b->fstat + g.Cp;
  BlockTrace& tr = b->trace;
  tr.reset(7 * d.m + 1);
  if (!eval) {
    {
      LaunchScope ls(b, KC_STATS, M * d.c0 * Sb, 0, M * d.c0 * 2.0);
      launch(k_channel_partials<S>, dim3(g.P, static_cast<unsigned>((d.c0 + 31) / 32)), 256, 0, b->stream, feat,
             static_cast<int>(g.Cp), 0, g.M, d.c0, b->part);
    }
    LaunchScope ls(b, KC_FINALIZE, 16.0 * g.P * d.c0, 0, 16.0 * g.P * d.c0);
    launch_finalize_stats_at(b->stream, b->part, g.P, d.c0, count, fmean, fvar, 0);
  }
  for (int l = 0; l < d.m; ++l) {
    LayerArgs<S> a = layer_args<S>(b, params, l);
    if (eval) {
      // every BN normalises with its own running statistics (ops.hpp:196-199)
      const float* r = running + b->stat_off[l];
      a.amean = r;
      a.avar = r + a.c;
      a.bmean = r + 2 * a.c;
      a.bvar = r + 2 * a.c + d.bk;
    }
    // trace (ops.hpp:565-595 conventions): the concat is a zero-copy channel
    // prefix (no moves: 0 FLOPs); BN_a + ReLU run in the 1x1 forward's transform
    tr.on(0, 7 * l + 0, BlockTrace::kConcat, 0.0);
    tr.on(0, 7 * l + 1, BlockTrace::kBatchNorm, 8.0 * M * a.c);
    tr.on(0, 7 * l + 2, BlockTrace::kRelu, M * a.c);
    tr.on(0, 7 * l + 3, BlockTrace::kConv, 2.0 * M * d.bk * a.c);
    tr.on(0, 7 * l + 4, BlockTrace::kBatchNorm, 8.0 * M * d.bk);
    tr.on(0, 7 * l + 5, BlockTrace::kRelu, M * d.bk);
    tr.on(0, 7 * l + 6, BlockTrace::kConv, 2.0 * M * d.k * 9.0 * d.bk);
    int p1 = g.P;  // BN_b partial rows
    {
      LaunchScope ls(b, KC_C1_FWD, M * (a.c + d.bk) * Sb, 2.0 * M * a.c * d.bk, M * (a.c + d.bk) * 2.0);
      if (b->tc) {
        if (!tc2_conv1x1_fwd(b, a, l, &p1)) tc_conv1x1_fwd(b, a);
      }
      else gemm_bn<128, Conv1x1Fwd>(b, a, g.M, d.bk, 1);
    }
    if (!eval) {
      LaunchScope ls(b, KC_FINALIZE, 16.0 * p1 * d.bk, 0, 16.0 * p1 * d.bk);
      float* zm = b->zstat + static_cast<int64_t>(l) * 2 * d.bk;
      launch_finalize_stats_at(b->stream, b->part, p1, d.bk, count, zm, zm + d.bk, 0);
    }
    int p3 = g.P;
    {
      LaunchScope ls(b, KC_C3_FWD, M * (d.bk + d.k) * Sb, 2.0 * M * 9 * d.bk * d.k, M * (d.bk + d.k) * 2.0);
      if (b->tc) p3 = tc_conv3x3_fwd(b, a, l);
      else gemm_bn<128, Conv3x3Fwd>(b, a, g.M, d.k, 1);
    }
    if (!eval) {
      LaunchScope ls(b, KC_FINALIZE, 16.0 * p3 * d.k, 0, 16.0 * p3 * d.k);
      launch_finalize_stats_at(b->stream, b->part, p3, d.k, count, fmean, fvar, a.c);
    }
  }
  tr.on(0, 7 * d.m, BlockTrace::kConcat, 0.0);  // block-output concat: the feature buffer itself
  if (!eval && update_running) {
    LaunchScope ls(b, KC_RUNNING, 0, 0, 0);
    launch(k_running_update, blocks_for(b->sz.stat_elems, 256), 256, 0, b->stream, 
        d.m, d.c0, d.k, d.bk, static_cast<int>(g.Cp), b->fstat, b->zstat, running,
        b->sz.stat_elems);
  }
}

template <typename S>
static void backward_impl(Block* b, const float* params, float* grad_acc, float* grads) {
  const dpb_block_desc& d = b->d;
  const Geometry& g = b->g;
  const int64_t hw = d.h * d.w;
  const double M = static_cast<double>(g.M), Sb = g.S;
  const double count = M;
  if (d.layout == DPB_NCHW) {
    LaunchScope ls(b, KC_PACK, M * g.C * 8, 0, M * g.C * 8);
    b->acc_cur = b->acc;
    dim3 grid(blocks_for(hw, 32), blocks_for(g.C, 32), static_cast<unsigned>(d.n));
    launch(k_nchw_to_nhwc<float>, grid, dim3(32, 8), 0, b->stream, grad_acc, d.n, g.C, hw,
                                                               b->acc, static_cast<int>(g.Cp), 0);
  } else {
    b->acc_cur = grad_acc;
  }
  if (b->tc) {
    LaunchScope ls(b, KC_PACK, 0, 0, 0);
    b->launches--;
    tc_pretile_w2(b, params, false);  // each pretile counts its own launch
    tc2_pretile_w1t(b, params);
  }
  // Two streams: the data-gradient chain (3x3 dgrad -> BN_b bwd -> 1x1 dgrad
  // -> BN_a bwd + accumulate) on the main stream, the weight-gradient branch
  // (3x3 wgrad -> fold, 1x1 wgrad -> fold) on the side stream.  g0 and the BN_b
  // coefficients are double-buffered by layer parity, so the side branch of
  // layer l overlaps the main chain of layers l and l-1.
  // DPB_NO_FORK=1 (debugging aid) keeps the whole backward on one stream.
  static const bool no_fork = std::getenv("DPB_NO_FORK") != nullptr;
  const bool fork = b->side != nullptr && !b->prof && !no_fork;
  cudaStream_t main_st = b->stream;
  auto ev = [&](int l, int which) { return b->fork_ev[3 * l + which]; };
  // split_apply: the accumulate's tail on side2 (DPB_NO_SPLIT_APPLY=1: off)
  static const bool no_split = std::getenv("DPB_NO_SPLIT_APPLY") != nullptr;
  const bool split = fork && b->side2 != nullptr && !no_split && d.k % 4 == 0 && d.c0 % 4 == 0 && d.m > 1;
  auto aev = [&](int l, int which) { return b->apply_ev[2 * l + which]; };
  for (int l = d.m - 1; l >= 0; --l) {
    LayerArgs<S> a = layer_args<S>(b, params, l);
    a.g0 = b->g0 + (l & 1) * g.M * d.bk;
    a.bnb_bwd = b->bnb_bwd + (l & 1) * 2 * d.bk;
    float* gl = grads + b->param_off[l];
    float* d_ga = gl;
    float* d_ba = gl + a.c;
    float* d_w1 = gl + 2 * a.c;
    float* d_gb = d_w1 + static_cast<int64_t>(d.bk) * a.c;
    float* d_bb = d_gb + d.bk;
    float* d_w2 = d_bb + d.bk;
    const double f3 = 2.0 * M * 9 * d.bk * d.k, f1 = 2.0 * M * a.c * d.bk;
    {
      // trace: the 3x3 dgrad prologue and the 3x3 wgrad each recompute act_b =
      // relu(bn_b(z)) (the mask, the operand); the 1x1 dgrad epilogue and the
      // 1x1 wgrad each recompute act_a (mask, operand) from the feature prefix
      // (graph.hpp:856-945 does it once, into Shared1/Shared2); conv backward
      // = dgrad + wgrad at 2x the forward FLOPs; the accumulate is the concat
      // backward (one add per element)
      BlockTrace& tr = b->trace;
      const double Mc = M * a.c, Mb = M * d.bk;
      for (int rep = 0; rep < 2; ++rep) {
        tr.on(2, 7 * l + 4, BlockTrace::kBatchNorm, 8.0 * Mb);
        tr.on(2, 7 * l + 5, BlockTrace::kRelu, Mb);
        tr.on(2, 7 * l + 1, BlockTrace::kBatchNorm, 8.0 * Mc);
        tr.on(2, 7 * l + 2, BlockTrace::kRelu, Mc);
      }
      tr.on(1, 7 * l + 6, BlockTrace::kConv, 2.0 * f3);
      tr.on(1, 7 * l + 5, BlockTrace::kRelu, Mb);
      tr.on(1, 7 * l + 4, BlockTrace::kBatchNorm, 12.0 * Mb);
      tr.on(1, 7 * l + 3, BlockTrace::kConv, 2.0 * f1);
      tr.on(1, 7 * l + 2, BlockTrace::kRelu, Mc);
      tr.on(1, 7 * l + 1, BlockTrace::kBatchNorm, 12.0 * Mc);
      tr.on(1, 7 * l + 0, BlockTrace::kConcat, Mc);
    }
    if (fork) {
      if (l + 2 < d.m) cudaStreamWaitEvent(main_st, ev(l + 2, 2), 0);  // buffers of parity l
      cudaEventRecord(ev(l, 0), main_st);
      cudaStreamWaitEvent(b->side, ev(l, 0), 0);
    }
    // ---- weight branch, part 1: 3x3 wgrad (graph.hpp:905-907) ----
    if (fork) b->stream = b->side;
    {
      const int64_t rows = 9LL * d.bk;
      int splits;
      {
        LaunchScope ls(b, KC_C3_WGRAD, M * (4.0 * d.k + Sb * d.bk), f3, M * (4.0 * d.k + 2.0 * d.bk));
        if (b->tc) {
          splits = tc_conv3x3_wgrad(b, a);
        } else {
          const int bn = bn_tile(d.k);
          const int64_t tiles = ((rows + 127) / 128) * ((d.k + bn - 1) / bn);
          a.kchunk = wgrad_chunk(g.M, tiles);
          splits = static_cast<int>((g.M + a.kchunk - 1) / a.kchunk);
          gemm_bn<128, Conv3x3Wgrad>(b, a, rows, d.k, splits);
        }
      }
      LaunchScope ls(b, KC_REDUCE_W, 4.0 * splits * rows * d.k, 0, 4.0 * splits * rows * d.k);
      launch(k_reduce_w2, blocks_for(9LL * d.k * d.bk, 32), dim3(32, 8), 0, b->stream, 
          b->wpart, splits, d.bk, d.k, d_w2);
    }
    b->stream = main_st;
    // ---- data chain: 3x3 dgrad (+ReLU mask by act_b, BN_b sums) ----
    int pd = g.P;
    {
      LaunchScope ls(b, KC_C3_DGRAD, M * (4.0 * d.k + Sb * d.bk + 4.0 * d.bk), f3, M * (4.0 * d.k + 2.0 * d.bk + 4.0 * d.bk));
      if (b->tc) pd = tc_conv3x3_dgrad(b, a, l);
      else gemm_bn<128, Conv3x3Dgrad>(b, a, g.M, d.bk, 1);
    }
    // BN_b backward sums -> dgamma_b, dbeta_b, coefficients (graph.hpp:913-916)
    {
      LaunchScope ls(b, KC_FINALIZE, 16.0 * pd * d.bk, 0, 16.0 * pd * d.bk);
      launch_finalize_bn_bwd(b->stream, b->part, pd, d.bk, count, d_gb, d_bb, const_cast<float*>(a.bnb_bwd));
    }
    if (fork) {
      cudaEventRecord(ev(l, 1), main_st);
      cudaStreamWaitEvent(b->side, ev(l, 1), 0);
    }
    // ---- weight branch, part 2: 1x1 wgrad (graph.hpp:920-922) ----
    if (fork) b->stream = b->side;
    {
      int splits;
      bool v2 = false;  // v2 partials are [split][j][i] like the SIMT ones
      {
        LaunchScope ls(b, KC_C1_WGRAD, M * ((4.0 + Sb) * d.bk + Sb * a.c), f1, M * ((4.0 + 2.0) * d.bk + 2.0 * a.c));
        if (b->tc) {
          splits = tc2_conv1x1_wgrad(b, a);
          v2 = splits > 0;
          if (!v2) splits = tc_conv1x1_wgrad(b, a);
        } else {
          const int64_t tiles = ((d.bk + 63) / 64) * ((a.c + 63) / 64);
          a.kchunk = wgrad_chunk(g.M, tiles);
          splits = static_cast<int>((g.M + a.kchunk - 1) / a.kchunk);
          gemm_bn2<64, Conv1x1Wgrad>(b, a, d.bk, a.c, splits);
        }
      }
      LaunchScope ls(b, KC_REDUCE_W, 4.0 * splits * d.bk * a.c, 0, 4.0 * splits * d.bk * a.c);
      if (b->tc && !v2)
        launch(k_reduce_w1t, blocks_for(static_cast<int64_t>(d.bk) * a.c, 32), dim3(32, 8), 0, b->stream, b->wpart, splits, d.bk, a.c, d_w1);
      else
        launch(k_reduce_w1, blocks_for(static_cast<int64_t>(d.bk) * a.c, 32), dim3(32, 8), 0, b->stream, b->wpart, splits, d.bk, a.c, d_w1);
    }
    if (fork) cudaEventRecord(ev(l, 2), b->side);
    b->stream = main_st;
    // the tail accumulate of layer l+2 read this layer's g1 / coefficient buffers
    if (split && l + 2 < d.m) cudaStreamWaitEvent(main_st, aev(l + 2, 1), 0);
    // ---- data chain: 1x1 dgrad (+ReLU mask by act_a, BN_a sums) ----
    {
      LaunchScope ls(b, KC_C1_DGRAD, M * ((4.0 + Sb) * d.bk + (Sb + 4.0) * a.c), f1, M * ((4.0 + 2.0) * d.bk + (2.0 + 4.0) * a.c));
      if (b->tc) {
        if (!tc2_conv1x1_dgrad(b, a, l)) tc_conv1x1_dgrad(b, a);
      }
      else gemm_bn2<128, Conv1x1Dgrad>(b, a, g.M, a.c, 1);
    }
    // BN_a backward (graph.hpp:929-932) + concat-backward accumulate (:936-941)
    float* bna = b->bna_bwd + (l & 1) * 2 * g.cmaxp;  // parity buffer (split_apply)
    {
      LaunchScope ls(b, KC_FINALIZE, 16.0 * g.P * a.c, 0, 16.0 * g.P * a.c);
      launch_finalize_bn_bwd(b->stream, b->part, g.P, a.c, count, d_ga, d_ba, bna);
    }
    // The accumulate of layer l updates channels [0, c_l); only its last k,
    // [c_l - k, c_l), feed layer l-1's 3x3 dgrad next.  With split_apply that
    // head runs on the main chain and the tail [0, c_l - k) on side2,
    // overlapping layer l-1's dgrads; per channel the accumulation order is
    // unchanged (tail l precedes head / tail l-1 through events), so results
    // are bit-identical to one accumulate per layer.
    const int c_head = (split && l > 0) ? a.c - d.k : 0;
    auto apply = [&](int c_lo, int c_hi, cudaStream_t st) {
      if (c_hi <= c_lo) return;
      LaunchScope ls(b, KC_BN_APPLY_ACC, M * (c_hi - c_lo) * (4.0 + Sb + 8.0), 0,
                     M * (c_hi - c_lo) * (4.0 + 2.0 + 8.0));
      const bool quads = std::is_same<S, float>::value && a.Ca % 4 == 0 && c_lo % 4 == 0 &&
                         (reinterpret_cast<uintptr_t>(b->acc_cur) & 15) == 0;
      const int nq = (c_hi + 3) / 4 - c_lo / 4;
      const bool narrow = nq <= 16;  // <= 64 channels: the main-chain head
      const int rows = narrow ? kApplyRowsNarrow : kApplyRows;
      if (quads)
        launch(narrow ? k_bn_apply_accumulate4<kApplyRowsNarrow> : k_bn_apply_accumulate4<kApplyRows>,
               blocks_for((g.M + rows - 1) / rows * nq, 256), 256, 0, st, g.M, c_lo, c_hi, a.C, a.Ca, a.cg,
               static_cast<const float*>(b->feat), a.g1, a.amean, a.avar, a.gamma_a,
               static_cast<const float*>(bna), b->acc_cur);
      else
        launch(k_bn_apply_accumulate<S>, blocks_for(g.M * (c_hi - c_lo), 256), 256, 0, st, g.M, c_lo, c_hi, a.C,
               a.Ca, a.cg, static_cast<const S*>(b->feat), a.g1, a.amean, a.avar, a.gamma_a,
               static_cast<const float*>(bna), b->acc_cur);
    };
    if (split) {
      cudaEventRecord(aev(l, 0), main_st);                                   // g1 + coefficients of layer l
      if (l + 1 < d.m) cudaStreamWaitEvent(main_st, aev(l + 1, 1), 0);      // tail of layer l+1
    }
    apply(c_head, a.c, main_st);
    if (split && l > 0) {
      cudaStreamWaitEvent(b->side2, aev(l, 0), 0);
      b->stream = b->side2;
      apply(0, c_head, b->side2);
      b->stream = main_st;
      cudaEventRecord(aev(l, 1), b->side2);
    }
  }
  if (fork) {  // join: the caller's stream sees every weight gradient
    cudaStreamWaitEvent(main_st, ev(0, 2), 0);
    if (d.m > 1) cudaStreamWaitEvent(main_st, ev(1, 2), 0);
  }
  if (d.layout == DPB_NCHW) {
    LaunchScope ls(b, KC_PACK, M * g.C * 8, 0, M * g.C * 8);
    dim3 grid(blocks_for(hw, 32), blocks_for(g.C, 32), static_cast<unsigned>(d.n));
    launch(k_nhwc_to_nchw<float>, grid, dim3(32, 8), 0, b->stream, b->acc, static_cast<int>(g.Cp), 0,
                                                               d.n, g.C, hw, grad_acc);
  }
}

// Folds shared with the whole-network step (dpb_model.cu).
// Many partial rows (the 56x56 blocks, the stem): 4 channels per CTA, so four
// times the CTAs share the fold.
constexpr int kFinWideP = 512;
void launch_finalize_bn_bwd(cudaStream_t st, const double2* part, int P, int nch, double count,
                            float* dgamma, float* dbeta, float* coef) {
  if (P > kFinWideP)
    launch(k_finalize_bn_bwd<4>, static_cast<unsigned>((nch + 3) / 4), kFinThreads, 0, st, part, P, nch, count,
           dgamma, dbeta, coef);
  else
    launch(k_finalize_bn_bwd<kFinCh>, static_cast<unsigned>((nch + kFinCh - 1) / kFinCh), kFinThreads, 0, st, part,
           P, nch, count, dgamma, dbeta, coef);
}
void launch_finalize_stats_at(cudaStream_t st, const double2* part, int P, int nch, double count, float* mean,
                              float* var, int first) {
  if (P > kFinWideP)
    launch(k_finalize_stats<4>, static_cast<unsigned>((nch + 3) / 4), kFinThreads, 0, st, part, P, nch, count, mean,
           var, first);
  else
    launch(k_finalize_stats<kFinCh>, static_cast<unsigned>((nch + kFinCh - 1) / kFinCh), kFinThreads, 0, st, part, P,
           nch, count, mean, var, first);
}
void launch_fold_splits(cudaStream_t st, const float* wpart, int splits, int64_t n, float* out) {
  launch(k_reduce_w1, blocks_for(n, 32), dim3(32, 8), 0, st, wpart, splits, 1, static_cast<int>(n), out);
}
void launch_channel_partials(cudaStream_t st, const float* src, int pitch, int64_t M, int nch, double2* part) {
  launch(k_channel_partials<float>, dim3(blocks_for(M, 128), static_cast<unsigned>((nch + 31) / 32)), 256, 0, st,
         src, pitch, 0, M, nch, part);
}
void launch_finalize_stats(cudaStream_t st, const double2* part, int P, int nch, double count, float* mean,
                           float* var) {
  launch_finalize_stats_at(st, part, P, nch, count, mean, var, 0);
}

int block_forward(Block* b, const float* x_in, const float* params, float* running,
                  int update_running, int eval) {
  if (b->g.M < 2 && !eval)
    return fail(DPB_DEGENERATE_BATCH_ERROR,
                "train-mode batchnorm needs at least 2 values per channel");
  if (eval && running == nullptr) return fail(DPB_CONFIG_ERROR, "eval needs running stats");
  b->launches = 0;
  forward_impl<float>(b, x_in, params, running, update_running, eval);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "block forward launch");
  b->fwd_done = !eval;
  return DPB_OK;
}

int block_backward(Block* b, const float* params, float* grad_acc, float* grads, int64_t acc_pitch) {
  if (!b->fwd_done)
    return fail(DPB_PROTOCOL_ERROR, "backward requires a train-mode forward");
  if (b->d.layout == DPB_NHWC && acc_pitch > 0 && acc_pitch < b->g.C)
    return fail(DPB_SHAPE_ERROR, "accumulator pitch below the block's channel count");
  // NCHW callers: the arena accumulator (pitch Cp); NHWC callers: their buffer
  b->acc_pitch = b->d.layout == DPB_NCHW ? b->g.Cp : (acc_pitch > 0 ? acc_pitch : b->g.C);
  b->launches = 0;
  backward_impl<float>(b, params, grad_acc, grads);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "block backward launch");
  return DPB_OK;
}

template <typename S>
static void read_feats_impl(Block* b, float* dst) {
  const dim3 grid(blocks_for(b->d.h * b->d.w, 32), blocks_for(b->g.C, 32),
                  static_cast<unsigned>(b->d.n));
  launch(k_nhwc_to_nchw<S>, grid, dim3(32, 8), 0, b->stream, 
      static_cast<const S*>(b->feat), static_cast<int>(b->g.Cp), 0, b->d.n,
      static_cast<int>(b->g.C), b->d.h * b->d.w, dst);
}

template <typename S>
static void read_z_impl(Block* b, float* dst) {
  const int64_t hw = b->d.h * b->d.w;
  const dim3 grid(blocks_for(hw, 32), blocks_for(b->d.bk, 32), static_cast<unsigned>(b->d.n));
  for (int l = 0; l < b->d.m; ++l)
    launch(k_nhwc_to_nchw<S>, grid, dim3(32, 8), 0, b->stream, 
        static_cast<const S*>(b->z) + static_cast<int64_t>(l) * b->g.M * b->d.bk, b->d.bk, 0,
        b->d.n, b->d.bk, hw, dst + static_cast<int64_t>(l) * b->g.M * b->d.bk);
}

int read_feats(Block* b, float* dst) {
  read_feats_impl<float>(b, dst);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DPB_OK : cuda_fail(e, "read_feats");
}

int read_z(Block* b, float* dst) {
  read_z_impl<float>(b, dst);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DPB_OK : cuda_fail(e, "read_z");
}

int read_stats(Block* b, float* dst) {
  launch(k_export_stats, blocks_for(b->sz.stat_elems, 256), 256, 0, b->stream, 
      b->d.m, b->d.c0, b->d.k, b->d.bk, static_cast<int>(b->g.Cp), b->fstat, b->zstat, dst,
      b->sz.stat_elems);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DPB_OK : cuda_fail(e, "read_stats");
}

int create(const dpb_block_desc* desc, int device, void* stream, Block** out, DeviceTracker* tracker) {
  int rc = validate(desc);
  if (rc) return rc;
  if (out == nullptr) return fail(DPB_CONFIG_ERROR, "null output handle");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  Block* b = new (std::nothrow) Block();
  if (!b) return fail(DPB_CAPACITY_ERROR, "host allocation failed");
  b->d = *desc;
  b->device = device;
  b->stream = static_cast<cudaStream_t>(stream);
  b->g = geometry(*desc);
  b->tc = desc->dtype == DPB_BF16 && tc_supported(*desc);
  plan_arena(*desc, &b->sz);
  e = cudaMalloc(&b->arena, static_cast<size_t>(b->sz.total_bytes));
  if (e != cudaSuccess) {
    delete b;
    return cuda_fail(e, "arena cudaMalloc");
  }
  if (tracker) b->tracker = tracker;
  {
    const dpb_arena_sizes& z = b->sz;
    const int64_t owned = z.feat_bytes + z.z_bytes + z.stats_bytes, grad = z.acc_bytes + z.g0_bytes + z.g1_bytes;
    b->tracker->alloc(DPB_ARENA_FEATURE_OWNED, owned);
    b->tracker->alloc(DPB_ARENA_SHARED_GRAD, grad);
    b->tracker->alloc(DPB_ARENA_SCRATCH, z.total_bytes - owned - grad);  // partials, weight images, alignment
  }
  char* base = static_cast<char*>(b->arena);
  b->feat = base + b->sz.feat_offset;
  b->z = base + b->sz.z_offset;
  b->fstat = reinterpret_cast<float*>(base + b->sz.stats_offset);
  b->zstat = b->fstat + 2 * b->g.Cp;
  b->acc = reinterpret_cast<float*>(base + b->sz.acc_offset);
  b->g0 = reinterpret_cast<float*>(base + b->sz.g0_offset);
  b->g1 = reinterpret_cast<float*>(base + b->sz.g1_offset);
  char* sc = base + b->sz.scratch_offset;
  b->part = reinterpret_cast<double2*>(sc);
  const int64_t pbytes =
      align_up(std::max<int64_t>(static_cast<int64_t>(b->g.Pmax) * std::max<int64_t>(b->g.C, desc->bk) * 16,
                                 zsplit_bytes(*desc) > 0 ? (b->g.M + 31) / 32 * desc->bk * 16 : 0), 256);
  b->wpart = reinterpret_cast<float*>(sc + pbytes);
  // wgrad partial region size = scratch - pbytes - coef region
  const int64_t coef_bytes = align_up((4LL * desc->bk + 4 * b->g.cmaxp) * 4, 256);
  const int64_t wt_bytes = b->tc ? weight_image_bytes(*desc) : 0;
  const int64_t zs_bytes = align_up(zsplit_bytes(*desc), 256);
  b->bnb_bwd = reinterpret_cast<float*>(sc + b->sz.scratch_bytes - wt_bytes - zs_bytes - coef_bytes);
  if (zs_bytes) b->zpart = reinterpret_cast<float*>(sc + b->sz.scratch_bytes - wt_bytes - zs_bytes);
  b->bna_bwd = b->bnb_bwd + 4 * desc->bk;
  if (b->tc) {
    // the pre-tiled weight images follow the scratch partials/coefficients
    b->halo = tc_halo_plan(*desc);
    uint8_t* wbase = reinterpret_cast<uint8_t*>(sc + b->sz.scratch_bytes - wt_bytes);
    int64_t w1 = 0;
    for (int l = 0; l < desc->m; ++l) {
      b->wtile_off.push_back(w1);
      w1 += tc2_w1_tile_bytes(*desc, l);
    }
    if (w1 > 0) b->wtile = wbase;
    uint8_t* p = wbase + align_up(w1, 256);
    if (b->halo.fwd_ok) b->w2f = p;
    p += align_up(b->halo.fwd_layer_bytes * desc->m, 256);
    if (b->halo.bwd_ok) b->w2b = p;
    p += align_up(b->halo.bwd_layer_bytes * desc->m, 256);
    int64_t w1b = 0;
    for (int l = 0; l < desc->m; ++l) {
      b->w1b_off.push_back(w1b);
      w1b += tc2_w1b_layer_bytes(*desc, l);
    }
    if (w1b > 0) b->w1b = p;
  }
  if (cudaStreamCreateWithFlags(&b->side, cudaStreamNonBlocking) != cudaSuccess) b->side = nullptr;
  if (b->side && cudaStreamCreateWithFlags(&b->side2, cudaStreamNonBlocking) != cudaSuccess) b->side2 = nullptr;
  for (int i = 0; b->side2 && i < 2 * desc->m; ++i) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    b->apply_ev.push_back(e);
  }
  for (int i = 0; b->side && i < 3 * desc->m; ++i) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    b->fork_ev.push_back(e);
  }
  int64_t po = 0, so = 0;
  for (int l = 0; l < desc->m; ++l) {
    const int64_t c = desc->c0 + static_cast<int64_t>(l) * desc->k;
    b->param_off.push_back(po);
    b->stat_off.push_back(so);
    po += 2 * c + desc->bk * c + 2LL * desc->bk + 9LL * desc->k * desc->bk;
    so += 2 * c + 2LL * desc->bk;
  }
  *out = b;
  return DPB_OK;
}

void destroy(Block* b) {
  if (!b) return;
  if (b->arena) {
    cudaFree(b->arena);
    const dpb_arena_sizes& z = b->sz;
    const int64_t owned = z.feat_bytes + z.z_bytes + z.stats_bytes, grad = z.acc_bytes + z.g0_bytes + z.g1_bytes;
    b->tracker->free(DPB_ARENA_FEATURE_OWNED, owned);
    b->tracker->free(DPB_ARENA_SHARED_GRAD, grad);
    b->tracker->free(DPB_ARENA_SCRATCH, z.total_bytes - owned - grad);
  }
  for (cudaEvent_t e : b->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : b->fork_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : b->apply_ev) cudaEventDestroy(e);
  if (b->side) cudaStreamDestroy(b->side);
  if (b->side2) cudaStreamDestroy(b->side2);
  delete b;
}

void profile_enable(Block* b, int on) {
  b->prof = on != 0;
  b->recs.clear();
  b->ev_used = 0;
}

int profile_read(Block* b, dpb_kernel_stat* out, int max, int* count) {
  const cudaError_t e = cudaStreamSynchronize(b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "profile sync");
  dpb_kernel_stat acc[KC_COUNT];
  std::memset(acc, 0, sizeof(acc));
  for (int c = 0; c < KC_COUNT; ++c)
    std::snprintf(acc[c].name, sizeof(acc[c].name), "%s", kKernelCatNames[c]);
  for (const ProfRec& r : b->recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.start, r.stop);
    acc[r.cat].launches++;
    acc[r.cat].total_ms += ms;
    acc[r.cat].bytes += r.bytes;
    acc[r.cat].flops += r.flops;
    acc[r.cat].bytes_8d += r.bytes_8d;
  }
  int n = 0;
  for (int c = 0; c < KC_COUNT && n < max; ++c)
    if (acc[c].launches) out[n++] = acc[c];
  *count = n;
  return DPB_OK;
}

}  // namespace dpb
