// Internal host-side types shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dpb.h"

namespace dpb {

// Exact device-byte accounting per arena (MemoryTracker, alloctrace.hpp:57-105):
// live / peak per ArenaTag and the combined feature peak (every arena but
// Params).  Every cudaMalloc of libdpb is recorded, split by the regions it
// holds; one tracker per model (its blocks record into it) or per block.
struct DeviceTracker {
  int64_t live[6] = {}, peak[6] = {};
  int64_t feature_live = 0, feature_peak = 0;
  void alloc(int tag, int64_t bytes) {
    live[tag] += bytes;
    if (live[tag] > peak[tag]) peak[tag] = live[tag];
    if (tag != DPB_ARENA_PARAMS) {
      feature_live += bytes;
      if (feature_live > feature_peak) feature_peak = feature_live;
    }
  }
  void free(int tag, int64_t bytes) {
    live[tag] -= bytes;
    if (tag != DPB_ARENA_PARAMS) feature_live -= bytes;
  }
  void snapshot(dpb_memory_stats* out) const {
    for (int i = 0; i < 6; ++i) {
      out->live_bytes[i] = live[i];
      out->peak_bytes[i] = peak[i];
    }
    out->total_feature_peak_bytes = feature_peak;
    out->param_bytes = live[DPB_ARENA_PARAMS];
  }
};

// OpTrace of the block (alloctrace.hpp:132-201): per-node forward / backward /
// recompute counts and per-OpKind FLOPs with the reference's conventions
// (ops.hpp:565-595), recorded by the host as the fused kernels run.  Nodes
// per layer l: 7l + {0 concat, 1 bn_a, 2 relu_a, 3 conv_a, 4 bn_b, 5 relu_b,
// 6 conv_b}; node 7m is the block-output concat.
struct BlockTrace {
  enum Kind { kConcat = 0, kBatchNorm = 1, kRelu = 2, kConv = 3, kKinds = 7 };
  std::vector<int32_t> counts;  // 3 per node: forward, backward, recompute
  double flops[3][kKinds] = {};
  void reset(int nodes) {
    counts.assign(3 * static_cast<size_t>(nodes), 0);
    for (auto& r : flops)
      for (double& f : r) f = 0.0;
  }
  void on(int what, int node, int kind, double f) {  // what: 0 fwd, 1 bwd, 2 recompute
    counts[3 * static_cast<size_t>(node) + what]++;
    flops[what][kind] += f;
  }
};

struct Geometry {
  int64_t M = 0;     // pixels N*H*W
  int64_t C = 0;     // block output channels c0 + m*k
  int64_t Cp = 0;    // feature-arena row pitch: C rounded up to 4 floats (16-byte rows for TMA)
  int64_t cmax = 0;  // widest layer input c0 + (m-1)*k
  int64_t cmaxp = 0; // cmax rounded up to 4 (g1 rows)
  int P = 0;         // row CTAs of 128 pixels = partial-sum count
  int Pmax = 0;      // partial rows allocated (>= P; halo kernels use N * tiles/image)
  int S = 4;         // bytes per stored feature element
};

// Kernel categories for the optional per-launch profiler (bench.py roofline).
enum KernelCat {
  KC_PACK = 0, KC_STATS, KC_FINALIZE, KC_C1_FWD, KC_C3_FWD, KC_C3_DGRAD, KC_C3_WGRAD,
  KC_C1_DGRAD, KC_C1_WGRAD, KC_REDUCE_W, KC_BN_APPLY_ACC, KC_RUNNING, KC_COUNT
};
extern const char* const kKernelCatNames[KC_COUNT];

struct ProfRec {
  int cat;
  cudaEvent_t start, stop;
  double bytes, flops;
  double bytes_8d;  // SURVEY 8(d) model bytes (bf16 activations, fp32 gradients)
};

// Tile choices of the 3x3 halo kernels (dpb_tc_block.cu tc_halo_plan).
struct HaloPlan {
  bool fwd_ok = false, bwd_ok = false;
  bool fwd_taps = false;  // forward as one GEMM over all 9 taps (Tc3x3FwdTaps)
  int fwd_bn = 0, fwd_kc = 0, bwd_bn = 0, bwd_kc = 0;
  int bwd_split = 1;  // 3x3 dgrad: output-column groups of bwd_bn per tile (grid.y)
  int fwd_ring = 2;   // 3x3 forward: raw halo ring depth (1 when that fits two CTAs per SM)
  int fwd_kpair = 0;  // 3x3 forward: K chunks split over a (1, 2) cluster per tile (few tiles)
  int64_t fwd_layer_bytes = 0, bwd_layer_bytes = 0;  // pre-tiled W2 image per layer
};

struct Block {
  dpb_block_desc d{};
  Geometry g;
  dpb_arena_sizes sz{};
  int device = 0;
  cudaStream_t stream = nullptr;
  void* arena = nullptr;
  DeviceTracker own_tracker;
  DeviceTracker* tracker = &own_tracker;  // the owning model's tracker when part of one
  void* feat = nullptr;      // [M, C] S
  void* z = nullptr;         // m x [M, bk] S
  float* fstat = nullptr;    // mean[C] | var[C]
  float* zstat = nullptr;    // per layer mean[bk] | var[bk]
  float* acc = nullptr;      // [M, C] fp32 (NCHW boundary only)
  float* acc_cur = nullptr;  // the accumulator in use (arena or caller NHWC)
  int64_t acc_pitch = 0;     // its row pitch (arena: Cp; caller NHWC: C or the caller's)
  float* g0 = nullptr;       // [M, bk] fp32 (x2: double-buffered across layers)
  cudaStream_t side = nullptr;        // weight-gradient branch of the backward
  std::vector<cudaEvent_t> fork_ev;   // per layer: start, bn_b done, side done
  cudaStream_t side2 = nullptr;       // the accumulate's tail (split apply)
  std::vector<cudaEvent_t> apply_ev;  // per layer: g1 ready, tail done
  float* g1 = nullptr;       // 2 x [M, cmax] fp32 (layer parity)
  double2* part = nullptr;   // per-CTA partial sums
  float* wpart = nullptr;    // split-K weight-gradient partials
  float* zpart = nullptr;    // split-K 1x1 forward partials [ks][M][bk] (null: no split)
  float* bnb_bwd = nullptr;  // [bk][2] (x2: double-buffered across layers)
  float* bna_bwd = nullptr;  // [cmax][2] (x2: layer parity)
  std::vector<int64_t> param_off, stat_off;
  uint8_t* wtile = nullptr;           // pre-tiled bf16 W1 operands (tensor-core path)
  std::vector<int64_t> wtile_off;
  HaloPlan halo;
  uint8_t* w1b = nullptr;             // pre-tiled W1^T (v2 1x1 dgrad), per layer
  std::vector<int64_t> w1b_off;
  uint8_t* w2f = nullptr;             // pre-tiled W2 (halo forward), per layer
  uint8_t* w2b = nullptr;             // pre-tiled W2^T (halo dgrad), per layer
  bool tc = false;                    // tensor-core (tcgen05) GEMMs
  bool fwd_done = false;
  int64_t launches = 0;
  bool prof = false;
  BlockTrace trace;                   // OpTrace of the last forward + backward
  std::vector<ProfRec> recs;          // recorded launches (profiling on)
  std::vector<cudaEvent_t> ev_pool;   // reusable events
  size_t ev_used = 0;
};

// Counts one kernel launch; when profiling is on, brackets it with CUDA
// events on the block's stream and records its algorithmic bytes / flops.
struct LaunchScope {
  Block* b;
  int idx = -1;
  int cat = 0;
  // bytes: algorithmic HBM bytes with this build's storage (fp32 features);
  // bytes_8d: the same traffic under SURVEY 8(d)'s model (2-byte activations)
  LaunchScope(Block* blk, int cat, double bytes, double flops, double bytes_8d);
  ~LaunchScope();
};

extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int validate(const dpb_block_desc* d);
Geometry geometry(const dpb_block_desc& d);
void plan_arena(const dpb_block_desc& d, dpb_arena_sizes* s);
int create(const dpb_block_desc* desc, int device, void* stream, Block** out,
           DeviceTracker* tracker = nullptr);
void destroy(Block* b);
int block_forward(Block* b, const float* x_in, const float* params, float* running,
                  int update_running, int eval);
// acc_pitch: row pitch of an NHWC grad_acc (<= 0: the block's C)
int block_backward(Block* b, const float* params, float* grad_acc, float* grads, int64_t acc_pitch = 0);
int read_feats(Block* b, float* dst);
int read_z(Block* b, float* dst);
int read_stats(Block* b, float* dst);
void profile_enable(Block* b, int on);
void launch_finalize_bn_bwd(cudaStream_t st, const double2* part, int P, int nch, double count,
                            float* dgamma, float* dbeta, float* coef);
void launch_fold_splits(cudaStream_t st, const float* wpart, int splits, int64_t n, float* out);
// fp64 per-128-row partial sums of an NHWC fp32 buffer and their fold into
// mean / biased variance (the block's statistics kernels, dpb_kernels.cuh)
void launch_channel_partials(cudaStream_t st, const float* src, int pitch, int64_t M, int nch, double2* part);
void launch_finalize_stats(cudaStream_t st, const double2* part, int P, int nch, double count, float* mean,
                           float* var);
void launch_finalize_stats_at(cudaStream_t st, const double2* part, int P, int nch, double count, float* mean,
                              float* var, int first);
int profile_read(Block* b, dpb_kernel_stat* out, int max, int* count);

// tensor-core path (dpb_tc_block.cu)
template <typename S>
struct LayerArgs;
bool tc_supported(const dpb_block_desc& d);
int64_t tc_wgrad_chunk(int64_t M, int64_t tiles);
void tc_conv1x1_fwd(Block* b, const LayerArgs<float>& a);
int tc_conv3x3_fwd(Block* b, const LayerArgs<float>& a, int l);    // returns partial rows
int tc_conv3x3_dgrad(Block* b, const LayerArgs<float>& a, int l);  // returns partial rows
HaloPlan tc_halo_plan(const dpb_block_desc& d);
void tc_pretile_w2(Block* b, const float* params, bool fwd);
int64_t tc_halo_partials(const dpb_block_desc& d);
int64_t tc_halo_wgrad_splits(const dpb_block_desc& d);
void tc_conv1x1_dgrad(Block* b, const LayerArgs<float>& a);
int tc_conv1x1_wgrad(Block* b, LayerArgs<float> a);
// prows: BN_b partial rows written (left unchanged = the 128-row tile count)
bool tc2_conv1x1_fwd(Block* b, const LayerArgs<float>& a, int l, int* prows = nullptr);
int tc2_fwd_ksplit(int64_t M, int c, int sms, int ns);
int64_t tc2_w1_tile_bytes(const dpb_block_desc& d, int l);
void tc2_pretile_w1(Block* b, const float* params);
int tc2_bwd_bn(const dpb_block_desc& d);
int64_t tc2_w1b_layer_bytes(const dpb_block_desc& d, int l);
void tc2_pretile_w1t(Block* b, const float* params);
bool tc2_conv1x1_dgrad(Block* b, const LayerArgs<float>& a, int l);
int64_t tc2_wgrad_wpart_elems(const dpb_block_desc& d, int l);
int tc2_conv1x1_wgrad(Block* b, const LayerArgs<float>& a);
int tc_conv3x3_wgrad(Block* b, LayerArgs<float> a);

}  // namespace dpb

