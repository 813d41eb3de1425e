// denseplan_b200/block.hpp — C++ host API over the dpb C ABI, mirroring the
// reference's dense-block surface (namespace denseplan, /root/reference/proj/
// include/denseplan): the error hierarchy (errors.hpp:8-61), Shape4
// (tensor.hpp:15-45), ArenaTag / MemoryStats accounting (alloctrace.hpp:17-105),
// and a BlockPlan that plays GraphPlan's dense-block role: build (graph.hpp:
// 405-613), forward (forward_layer loop, :618-670 / :747-760) and backward
// (backward_block / backward_layer with rematerialize, :1054-1063 / :856-945).
//
// Header-only; link with libdpb.so.  Device pointers are caller-owned (CUDA
// allocations); the plan owns its HBM arena.  Like GraphPlan the plan is
// move-only and single-threaded (alloctrace.hpp:55-56).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../dpb.h"

namespace denseplan_b200 {

// ---- errors.hpp:8-61, same names, thrown for the matching status code ----
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error { using Error::Error; };
struct BoundsError : Error { using Error::Error; };
struct SizeOverflowError : Error { using Error::Error; };
struct CapacityError : Error { using Error::Error; };
struct AccountingError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct LabelError : Error { using Error::Error; };
struct DegenerateBatchError : Error { using Error::Error; };
struct ProtocolError : Error { using Error::Error; };
struct RangeError : Error { using Error::Error; };
struct VerifyError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

inline void check(int status) {
  if (status == DPB_OK) return;
  const std::string msg = dpb_last_error();
  switch (status) {
    case DPB_SHAPE_ERROR: throw ShapeError(msg);
    case DPB_BOUNDS_ERROR: throw BoundsError(msg);
    case DPB_SIZE_OVERFLOW_ERROR: throw SizeOverflowError(msg);
    case DPB_CAPACITY_ERROR: throw CapacityError(msg);
    case DPB_ACCOUNTING_ERROR: throw AccountingError(msg);
    case DPB_CONFIG_ERROR: throw ConfigError(msg);
    case DPB_FORMAT_ERROR: throw FormatError(msg);
    case DPB_LABEL_ERROR: throw LabelError(msg);
    case DPB_DEGENERATE_BATCH_ERROR: throw DegenerateBatchError(msg);
    case DPB_PROTOCOL_ERROR: throw ProtocolError(msg);
    case DPB_RANGE_ERROR: throw RangeError(msg);
    case DPB_VERIFY_ERROR: throw VerifyError(msg);
    default: throw DeviceError(msg);
  }
}

// ---- tensor.hpp:15-45 ----------------------------------------------------
struct Shape4 {
  std::int64_t n = 0, c = 0, h = 0, w = 0;
  friend bool operator==(const Shape4&, const Shape4&) = default;
  bool valid() const { return n >= 1 && c >= 1 && h >= 1 && w >= 1; }
  std::int64_t elems() const {
    if (!valid()) throw ShapeError("invalid shape (" + str() + ")");
    unsigned __int128 p = static_cast<unsigned __int128>(n);
    p *= static_cast<unsigned __int128>(c);
    p *= static_cast<unsigned __int128>(h);
    p *= static_cast<unsigned __int128>(w);
    if (p > static_cast<unsigned __int128>(INT64_MAX / 16))
      throw SizeOverflowError("shape " + str() + " overflows element count");
    return static_cast<std::int64_t>(p);
  }
  std::string str() const {
    return std::to_string(n) + "x" + std::to_string(c) + "x" + std::to_string(h) + "x" +
           std::to_string(w);
  }
};

// ---- alloctrace.hpp:17-24 -----------------------------------------------------
enum class ArenaTag {
  Params = DPB_ARENA_PARAMS,
  FeatureOwned = DPB_ARENA_FEATURE_OWNED,
  Shared1 = DPB_ARENA_SHARED1,
  Shared2 = DPB_ARENA_SHARED2,
  SharedGrad = DPB_ARENA_SHARED_GRAD,
  Scratch = DPB_ARENA_SCRATCH,
};

enum class Precision { FP32 = DPB_FP32, BF16 = DPB_BF16 };
enum class Layout { NCHW = DPB_NCHW, NHWC = DPB_NHWC };

// Geometry of one dense block (densenet.hpp:124-180; bottleneck width 4k at :68).
struct BlockConfig {
  std::int64_t n = 0, h = 0, w = 0;
  int c0 = 0, layers = 0, growth_rate = 0, bottleneck = 0;
  Precision precision = Precision::BF16;
  Layout layout = Layout::NCHW;

  int c_out() const { return c0 + layers * growth_rate; }
  int c_in(int l) const { return c0 + l * growth_rate; }
  dpb_block_desc desc() const {
    dpb_block_desc d{};
    d.n = n;
    d.h = h;
    d.w = w;
    d.c0 = c0;
    d.m = layers;
    d.k = growth_rate;
    d.bk = bottleneck > 0 ? bottleneck : 4 * growth_rate;
    d.dtype = static_cast<int32_t>(precision);
    d.layout = static_cast<int32_t>(layout);
    return d;
  }
};

// Per-arena byte accounting of the plan (MemoryStats analogue): the shared
// forward pools the reference allocates (Shared1/Shared2) are 0 here because
// concat is a zero-copy channel prefix and BN+ReLU are recomputed in the
// convolution prologues.
struct ArenaPlan {
  dpb_arena_sizes raw{};
  std::int64_t bytes(ArenaTag tag) const {
    switch (tag) {
      case ArenaTag::FeatureOwned: return raw.feat_bytes + raw.z_bytes + raw.stats_bytes;
      case ArenaTag::Shared1: return raw.shared1_bytes;
      case ArenaTag::Shared2: return raw.shared2_bytes;
      case ArenaTag::SharedGrad: return raw.acc_bytes + raw.g0_bytes + raw.g1_bytes;
      case ArenaTag::Scratch: return raw.scratch_bytes;
      case ArenaTag::Params: return 0;  // caller-owned
    }
    return 0;
  }
  std::int64_t total() const { return raw.total_bytes; }
};

inline ArenaPlan plan_arena(const BlockConfig& cfg) {
  ArenaPlan p;
  const dpb_block_desc d = cfg.desc();
  check(dpb_block_plan(&d, &p.raw));
  return p;
}

// The dense-block share of GraphPlan<T> (graph.hpp:234-268): build once,
// then forward / backward per step.
class BlockPlan {
 public:
  static BlockPlan build(const BlockConfig& cfg, int device = 0, void* stream = nullptr) {
    BlockPlan p;
    p.cfg_ = cfg;
    const dpb_block_desc d = cfg.desc();
    check(dpb_block_create(&d, device, stream, &p.h_));
    check(dpb_block_param_elems(&d, &p.param_elems_, &p.stat_elems_));
    return p;
  }
  BlockPlan(BlockPlan&& o) noexcept { *this = std::move(o); }
  BlockPlan& operator=(BlockPlan&& o) noexcept {
    std::swap(h_, o.h_);
    cfg_ = o.cfg_;
    param_elems_ = o.param_elems_;
    stat_elems_ = o.stat_elems_;
    freeze_running_ = o.freeze_running_;
    return *this;
  }
  BlockPlan(const BlockPlan&) = delete;
  BlockPlan& operator=(const BlockPlan&) = delete;
  ~BlockPlan() {
    if (h_) dpb_block_destroy(h_);
  }

  const BlockConfig& config() const { return cfg_; }
  std::int64_t param_elems() const { return param_elems_; }
  std::int64_t stat_elems() const { return stat_elems_; }
  ArenaPlan arena() const {
    ArenaPlan a;
    check(dpb_block_arena(h_, &a.raw, nullptr));
    return a;
  }
  void set_stream(void* stream) { check(dpb_block_set_stream(h_, stream)); }

  // Train-mode forward (forward_layer loop); running stats updated with the
  // momentum rule unless frozen (set_freeze_running_stats, graph.hpp:254).
  void forward(const float* x_in, const float* params, float* running) {
    check(dpb_block_forward(h_, x_in, params, running, freeze_running_ ? 0 : 1));
  }
  void forward_eval(const float* x_in, const float* params, const float* running) {
    check(dpb_block_forward_eval(h_, x_in, params, running));
  }
  // backward_block: grad_acc in/out, grads written (graph.hpp:1054-1063).
  void backward(const float* params, float* grad_acc, float* grads) {
    check(dpb_block_backward(h_, params, grad_acc, grads));
  }
  void set_freeze_running_stats(bool freeze) { freeze_running_ = freeze; }

  void read_feats(float* dst) const { check(dpb_block_read_feats(h_, dst)); }
  void read_z(float* dst) const { check(dpb_block_read_z(h_, dst)); }
  void read_stats(float* dst) const { check(dpb_block_read_stats(h_, dst)); }
  void sync() const { check(dpb_sync(h_)); }
  std::int64_t launch_count() const { return dpb_block_launch_count(h_); }

 private:
  BlockPlan() = default;
  dpb_block* h_ = nullptr;
  BlockConfig cfg_{};
  std::int64_t param_elems_ = 0, stat_elems_ = 0;
  bool freeze_running_ = false;
};

// densenet.hpp:234-275 / peak_model.hpp:37-158 over the C ABI.
inline std::int64_t count_parameters(const std::vector<int32_t>& blocks, int k, bool bottleneck,
                                     double compression, int classes, int c0, int in_c = 3) {
  std::int64_t out = 0;
  check(dpb_count_parameters(static_cast<int>(blocks.size()), blocks.data(), k, bottleneck,
                             compression, classes, c0, in_c, &out));
  return out;
}

}  // namespace denseplan_b200
