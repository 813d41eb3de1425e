// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Thin extern "C" driver over the UNMODIFIED reference headers
// (/root/reference/proj/include/denseplan, header-only C++20).  Built by
// oracle/Makefile into oracle/_ref/libdenseplan_ref.so; never linked by the
// product.  Used to
//   (1) generate the golden vectors in tests/golden/ (oracle/gen_golden.py),
//   (2) pin the block-level harness below against GraphPlan::step_trace
//       bitwise (ref_check_block_harness), and
//   (3) time the reference CPU path for bench.py --impl reference.
//
// The block-level harness calls only the reference's PUBLIC ops:: functions,
// in exactly the order of GraphPlan::forward_layer (dp/graph.hpp:618-670)
// and backward_layer (dp/graph.hpp:856-945), with rematerialization from the
// saved statistics (dp/graph.hpp:831-854, 884-901).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "denseplan/densenet.hpp"
#include "denseplan/errors.hpp"
#include "denseplan/graph.hpp"
#include "denseplan/ops.hpp"
#include "denseplan/schedule.hpp"
#include "denseplan/train.hpp"
#include "denseplan/peak_model.hpp"
#include "denseplan/rng.hpp"
#include "denseplan/tensor.hpp"

using namespace denseplan;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError& e) { g_err = e.what(); return 1; }
  catch (const BoundsError& e) { g_err = e.what(); return 2; }
  catch (const SizeOverflowError& e) { g_err = e.what(); return 3; }
  catch (const CapacityError& e) { g_err = e.what(); return 4; }
  catch (const AccountingError& e) { g_err = e.what(); return 5; }
  catch (const ConfigError& e) { g_err = e.what(); return 6; }
  catch (const FormatError& e) { g_err = e.what(); return 7; }
  catch (const LabelError& e) { g_err = e.what(); return 8; }
  catch (const DegenerateBatchError& e) { g_err = e.what(); return 9; }
  catch (const ProtocolError& e) { g_err = e.what(); return 10; }
  catch (const RangeError& e) { g_err = e.what(); return 11; }
  catch (const VerifyError& e) { g_err = e.what(); return 12; }
  catch (const std::exception& e) { g_err = e.what(); return 99; }
}

template <typename T>
Tensor<T> from_flat(const T* src, const Shape4& s, MemoryTracker& tr) {
  Tensor<T> t = Tensor<T>::alloc(s, ArenaTag::Scratch, tr);
  std::memcpy(t.data(), src, sizeof(T) * static_cast<std::size_t>(s.elems()));
  return t;
}

template <typename T>
void to_flat(const Tensor<T>& t, T* dst) {
  const Shape4& s = t.shape();
  std::int64_t o = 0;
  for (std::int64_t i = 0; i < s.n; ++i)
    for (std::int64_t c = 0; c < s.c; ++c)
      for (std::int64_t y = 0; y < s.h; ++y)
        for (std::int64_t x = 0; x < s.w; ++x) dst[o++] = t.at(i, c, y, x);
}

template <typename T>
struct HLayer {
  ops::BatchNormState<T> bn_a, bn_b;
  ops::ConvParams<T> conv_a, conv_b;
  Tensor<T> d_ga, d_ba, d_w1, d_gb, d_bb, d_w2;
  Tensor<T> z, y;
  ops::BatchStats<T> stats_a, stats_b;
};

template <typename T>
ops::BatchNormState<T> make_bn(const T* g, const T* b, const T* rm,
                               const T* rv, std::int64_t c,
                               MemoryTracker& tr) {
  ops::BatchNormState<T> bn;
  bn.gamma = from_flat(g, Shape4{1, c, 1, 1}, tr);
  bn.beta = from_flat(b, Shape4{1, c, 1, 1}, tr);
  bn.running_mean.assign(rm, rm + c);
  bn.running_var.assign(rv, rv + c);
  return bn;
}

// Block-level harness over public ops:: (see file header).  Layouts are the
// flat ones documented in oracle/dp_oracle.c.
template <typename T>
void block_harness(std::int64_t n, std::int64_t h, std::int64_t w,
                   std::int64_t c0, std::int64_t m, std::int64_t k,
                   std::int64_t bk, const T* params, const T* x_in,
                   T* running, int update_running, T* feats_out, T* z_out,
                   T* stats_out, T* acc /* in/out, may be null */,
                   T* grads_out) {
  MemoryTracker tr;
  const std::int64_t c_out = c0 + m * k;
  std::vector<Tensor<T>> feats{from_flat(x_in, Shape4{n, c0, h, w}, tr)};
  std::vector<HLayer<T>> layers(static_cast<std::size_t>(m));
  std::int64_t po = 0, so = 0;
  for (std::int64_t l = 0; l < m; ++l) {
    const std::int64_t c = c0 + l * k;
    HLayer<T>& L = layers[static_cast<std::size_t>(l)];
    const T* ga = params + po;
    const T* ba = ga + c;
    const T* w1 = ba + c;
    const T* gb = w1 + bk * c;
    const T* bb = gb + bk;
    const T* w2 = bb + bk;
    T* rm_a = running + so;
    L.bn_a = make_bn(ga, ba, rm_a, rm_a + c, c, tr);
    L.bn_b = make_bn(gb, bb, rm_a + 2 * c, rm_a + 2 * c + bk, bk, tr);
    L.conv_a.weights = from_flat(w1, Shape4{bk, c, 1, 1}, tr);
    L.conv_a.padding = 0;
    L.conv_b.weights = from_flat(w2, Shape4{k, bk, 3, 3}, tr);
    L.conv_b.padding = 1;
    po += 2 * c + bk * c + 2 * bk + 9 * k * bk;
    so += 2 * c + 2 * bk;

    // forward_layer (graph.hpp:618-670)
    const Shape4 cat_shape{n, c, h, w};
    Tensor<T> cat = Tensor<T>::alloc(cat_shape, ArenaTag::Shared1, tr);
    ops::concat_forward(feats, cat);
    Tensor<T> a = Tensor<T>::alloc(cat_shape, ArenaTag::Shared2, tr);
    L.stats_a = ops::batchnorm_forward(cat, L.bn_a, ops::BnMode::Train, a,
                                       update_running != 0);
    ops::relu_inplace(a);
    const Shape4 mid{n, bk, h, w};
    L.z = Tensor<T>::alloc(mid, ArenaTag::FeatureOwned, tr);
    ops::conv2d_forward(a, L.conv_a, L.z);
    Tensor<T> a2 = Tensor<T>::alloc(mid, ArenaTag::Shared2, tr);
    L.stats_b = ops::batchnorm_forward(L.z, L.bn_b, ops::BnMode::Train, a2,
                                       update_running != 0);
    ops::relu_inplace(a2);
    L.y = Tensor<T>::alloc(Shape4{n, k, h, w}, ArenaTag::FeatureOwned, tr);
    ops::conv2d_forward(a2, L.conv_b, L.y);
    feats.push_back(L.y);
    // outputs
    to_flat(L.z, z_out + l * n * bk * h * w);
    T* st = stats_out + (so - 2 * c - 2 * bk);
    std::copy(L.stats_a.mean.begin(), L.stats_a.mean.end(), st);
    std::copy(L.stats_a.var.begin(), L.stats_a.var.end(), st + c);
    std::copy(L.stats_b.mean.begin(), L.stats_b.mean.end(), st + 2 * c);
    std::copy(L.stats_b.var.begin(), L.stats_b.var.end(), st + 2 * c + bk);
    T* rn = running + (so - 2 * c - 2 * bk);
    std::copy(L.bn_a.running_mean.begin(), L.bn_a.running_mean.end(), rn);
    std::copy(L.bn_a.running_var.begin(), L.bn_a.running_var.end(), rn + c);
    std::copy(L.bn_b.running_mean.begin(), L.bn_b.running_mean.end(), rn + 2 * c);
    std::copy(L.bn_b.running_var.begin(), L.bn_b.running_var.end(),
              rn + 2 * c + bk);
  }
  // block-output concat (graph.hpp:756-760)
  Tensor<T> out_cat = ops::concat_forward(feats, ArenaTag::Shared1, tr);
  to_flat(out_cat, feats_out);
  if (acc == nullptr) return;

  // backward_block (graph.hpp:1054-1063)
  Tensor<T> A = from_flat(acc, Shape4{n, c_out, h, w}, tr);
  std::vector<std::int64_t> poffs;
  {
    std::int64_t p = 0;
    for (std::int64_t l = 0; l < m; ++l) {
      poffs.push_back(p);
      const std::int64_t c = c0 + l * k;
      p += 2 * c + bk * c + 2 * bk + 9 * k * bk;
    }
  }
  for (std::int64_t l = m - 1; l >= 0; --l) {
    const std::int64_t c = c0 + l * k;
    HLayer<T>& L = layers[static_cast<std::size_t>(l)];
    const Shape4 cat_shape{n, c, h, w};
    const Shape4 mid{n, bk, h, w};
    Tensor<T> grad_out = A.channel_view(c, k);
    // rematerialize (graph.hpp:831-854) with the saved stats
    std::vector<Tensor<T>> ins(feats.begin(), feats.begin() + 1 + l);
    Tensor<T> cat = Tensor<T>::alloc(cat_shape, ArenaTag::Shared1, tr);
    ops::concat_forward(ins, cat);
    Tensor<T> act_a = Tensor<T>::alloc(cat_shape, ArenaTag::Shared2, tr);
    ops::batchnorm_apply(cat, L.bn_a, L.stats_a, act_a);
    ops::relu_inplace(act_a);
    Tensor<T> act_b = Tensor<T>::alloc(mid, ArenaTag::Shared2, tr);
    ops::batchnorm_apply(L.z, L.bn_b, L.stats_b, act_b);
    ops::relu_inplace(act_b);
    L.d_w2 = Tensor<T>::alloc(L.conv_b.weights.shape(), ArenaTag::Params, tr);
    L.d_w1 = Tensor<T>::alloc(L.conv_a.weights.shape(), ArenaTag::Params, tr);
    L.d_ga = Tensor<T>::alloc(Shape4{1, c, 1, 1}, ArenaTag::Params, tr);
    L.d_ba = Tensor<T>::alloc(Shape4{1, c, 1, 1}, ArenaTag::Params, tr);
    L.d_gb = Tensor<T>::alloc(Shape4{1, bk, 1, 1}, ArenaTag::Params, tr);
    L.d_bb = Tensor<T>::alloc(Shape4{1, bk, 1, 1}, ArenaTag::Params, tr);
    // graph.hpp:905-945
    Tensor<T> t0 = Tensor<T>::alloc(mid, ArenaTag::SharedGrad, tr);
    ops::conv2d_backward(grad_out, act_b, L.conv_b, &t0, L.d_w2);
    ops::relu_backward_inplace(t0, act_b);
    Tensor<T> t1 = Tensor<T>::alloc(mid, ArenaTag::SharedGrad, tr);
    ops::batchnorm_backward(t0, L.z, L.bn_b, L.stats_b, t1, L.d_gb, L.d_bb);
    Tensor<T> t2 = Tensor<T>::alloc(cat_shape, ArenaTag::SharedGrad, tr);
    ops::conv2d_backward(t1, act_a, L.conv_a, &t2, L.d_w1);
    ops::relu_backward_inplace(t2, act_a);
    Tensor<T> t3 = Tensor<T>::alloc(cat_shape, ArenaTag::SharedGrad, tr);
    ops::batchnorm_backward(t2, cat, L.bn_a, L.stats_a, t3, L.d_ga, L.d_ba);
    for (std::int64_t ch = 0; ch < c; ++ch)
      for (std::int64_t i = 0; i < n; ++i)
        for (std::int64_t y = 0; y < h; ++y)
          for (std::int64_t x = 0; x < w; ++x) A.at(i, ch, y, x) += t3.at(i, ch, y, x);
    T* g = grads_out + poffs[static_cast<std::size_t>(l)];
    to_flat(L.d_ga, g);
    to_flat(L.d_ba, g + c);
    to_flat(L.d_w1, g + 2 * c);
    to_flat(L.d_gb, g + 2 * c + bk * c);
    to_flat(L.d_bb, g + 2 * c + bk * c + bk);
    to_flat(L.d_w2, g + 2 * c + bk * c + 2 * bk);
  }
  to_flat(A, acc);
}

DenseNetConfig single_block_cfg(int m, int k, int c0, int classes) {
  return build_config({m}, k, true, 1.0, ActivationOrder::PreActivation,
                      classes, c0);
}

template <typename T>
Tensor<T> make_input(const Shape4& s, std::uint64_t seed, MemoryTracker& tr) {
  Tensor<T> t = Tensor<T>::alloc(s, ArenaTag::Scratch, tr);
  Rng rng(seed);
  for (std::int64_t i = 0; i < s.n; ++i)
    for (std::int64_t c = 0; c < s.c; ++c)
      for (std::int64_t y = 0; y < s.h; ++y)
        for (std::int64_t x = 0; x < s.w; ++x)
          t.at(i, c, y, x) = static_cast<T>(rng.normal());
  return t;
}

std::vector<int> make_labels(int n, int classes) {
  std::vector<int> l(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) l[static_cast<std::size_t>(i)] = i % classes;
  return l;
}

// Recomputes a single-block model's step with the block harness (stem and
// head via public ops::, as in graph.hpp:740-745, 787-826, 1088-1123,
// 1170-1181) and compares every parameter gradient and the loss BITWISE with
// GraphPlan<T>::step_trace.  Returns 0 on bitwise agreement, 12 otherwise.
template <typename T>
void check_block_harness(int m, int k, int c0, int n, int h, int w,
                         std::uint64_t seed) {
  const int classes = 4;
  const DenseNetConfig cfg = single_block_cfg(m, k, c0, classes);
  const Shape4 in{n, 3, h, w};
  MemoryTracker data_tr;
  Tensor<T> input = make_input<T>(in, seed + 99, data_tr);
  const std::vector<int> labels = make_labels(n, classes);
  GraphPlan<T> plan = GraphPlan<T>::build(cfg, ExecutionStrategy::SharedAll, in, seed);
  // snapshot params before the step (step_trace only touches grads/running)
  auto& P = plan.params();
  const std::int64_t bk = 4 * k;
  std::vector<T> flat;
  std::size_t idx = 1;  // params_[0] = stem.conv.w
  for (int l = 0; l < m; ++l)
    for (int j = 0; j < 6; ++j, ++idx) {
      const Tensor<T>& v = P[idx].value;
      const std::size_t off = flat.size();
      flat.resize(off + static_cast<std::size_t>(v.elems()));
      to_flat(v, flat.data() + off);
    }
  const StepResult<T> r = plan.step_trace(input, labels);

  // harness path
  MemoryTracker tr;
  ops::ConvParams<T> stem;
  stem.weights = P[0].value;
  stem.padding = 1;
  Tensor<T> stem_out = Tensor<T>::alloc(Shape4{n, c0, h, w}, ArenaTag::Scratch, tr);
  ops::conv2d_forward(input, stem, stem_out);
  std::vector<T> x_in(static_cast<std::size_t>(n) * c0 * h * w);
  to_flat(stem_out, x_in.data());
  std::int64_t stats_len = 0;
  for (int l = 0; l < m; ++l) stats_len += 2 * (c0 + l * k) + 2 * bk;
  std::vector<T> running(static_cast<std::size_t>(stats_len));
  {
    std::int64_t so = 0;
    for (int l = 0; l < m; ++l) {
      const std::int64_t c = c0 + l * k;
      std::fill(running.begin() + so, running.begin() + so + c, T(0));
      std::fill(running.begin() + so + c, running.begin() + so + 2 * c, T(1));
      std::fill(running.begin() + so + 2 * c, running.begin() + so + 2 * c + bk, T(0));
      std::fill(running.begin() + so + 2 * c + bk,
                running.begin() + so + 2 * c + 2 * bk, T(1));
      so += 2 * c + 2 * bk;
    }
  }
  const std::int64_t c_out = c0 + static_cast<std::int64_t>(m) * k;
  std::vector<T> feats(static_cast<std::size_t>(n * c_out * h * w));
  std::vector<T> z(static_cast<std::size_t>(m * n * bk * h * w));
  std::vector<T> stats(static_cast<std::size_t>(stats_len));
  // first a forward-only pass to get the block output for the head
  std::vector<T> running_copy = running;
  block_harness<T>(n, h, w, c0, m, k, bk, flat.data(), x_in.data(),
                   running_copy.data(), 1, feats.data(), z.data(), stats.data(),
                   nullptr, nullptr);
  // head forward (graph.hpp:787-809) + loss (815-826)
  const std::size_t hb = 1 + static_cast<std::size_t>(m) * 6;
  ops::BatchNormState<T> hbn;
  hbn.gamma = P[hb].value;
  hbn.beta = P[hb + 1].value;
  hbn.running_mean.assign(static_cast<std::size_t>(c_out), T(0));
  hbn.running_var.assign(static_cast<std::size_t>(c_out), T(1));
  const Shape4 hs{n, c_out, h, w};
  Tensor<T> cat = from_flat(feats.data(), hs, tr);
  Tensor<T> act = Tensor<T>::alloc(hs, ArenaTag::Scratch, tr);
  ops::BatchStats<T> hst = ops::batchnorm_forward(cat, hbn, ops::BnMode::Train, act);
  ops::relu_inplace(act);
  Tensor<T> gap = Tensor<T>::alloc(Shape4{n, c_out, 1, 1}, ArenaTag::Scratch, tr);
  ops::global_avgpool_forward(act, gap);
  Tensor<T> logits = Tensor<T>::alloc(Shape4{n, classes, 1, 1}, ArenaTag::Scratch, tr);
  ops::linear_forward(gap, P[hb + 2].value, P[hb + 3].value, logits);
  Tensor<T> glog = Tensor<T>::alloc(logits.shape(), ArenaTag::Scratch, tr);
  const T loss = ops::softmax_xent(logits, labels, glog);
  // head backward (graph.hpp:1088-1123)
  Tensor<T> g_gap = Tensor<T>::alloc(gap.shape(), ArenaTag::Scratch, tr);
  Tensor<T> gw = Tensor<T>::alloc(P[hb + 2].value.shape(), ArenaTag::Scratch, tr);
  Tensor<T> gb = Tensor<T>::alloc(P[hb + 3].value.shape(), ArenaTag::Scratch, tr);
  ops::linear_backward(glog, gap, P[hb + 2].value, g_gap, gw, gb);
  Tensor<T> g_act = Tensor<T>::alloc(hs, ArenaTag::Scratch, tr);
  ops::global_avgpool_backward(g_gap, g_act);
  ops::relu_backward_inplace(g_act, act);
  Tensor<T> acc = Tensor<T>::alloc(hs, ArenaTag::Scratch, tr);
  Tensor<T> dhg = Tensor<T>::alloc(Shape4{1, c_out, 1, 1}, ArenaTag::Scratch, tr);
  Tensor<T> dhb = Tensor<T>::alloc(Shape4{1, c_out, 1, 1}, ArenaTag::Scratch, tr);
  ops::batchnorm_backward(g_act, cat, hbn, hst, acc, dhg, dhb);
  std::vector<T> accv(static_cast<std::size_t>(n * c_out * h * w));
  to_flat(acc, accv.data());
  std::vector<T> grads(flat.size());
  block_harness<T>(n, h, w, c0, m, k, bk, flat.data(), x_in.data(),
                   running.data(), 1, feats.data(), z.data(), stats.data(),
                   accv.data(), grads.data());
  // stem wgrad (graph.hpp:1170-1181)
  Tensor<T> A = from_flat(accv.data(), hs, tr);
  Tensor<T> gstem = Tensor<T>::alloc(stem.weights.shape(), ArenaTag::Scratch, tr);
  ops::conv2d_backward(A.channel_view(0, c0), input, stem,
                       static_cast<Tensor<T>*>(nullptr), gstem);

  auto same = [](const Tensor<T>& a, const T* b) {
    std::vector<T> v(static_cast<std::size_t>(a.elems()));
    to_flat(a, v.data());
    return std::memcmp(v.data(), b, v.size() * sizeof(T)) == 0;
  };
  bool ok = std::memcmp(&loss, &r.loss, sizeof(T)) == 0;
  {
    std::vector<T> v(static_cast<std::size_t>(gstem.elems()));
    to_flat(gstem, v.data());
    ok = ok && same(P[0].grad, v.data());
  }
  std::size_t off = 0;
  idx = 1;
  for (int l = 0; l < m; ++l)
    for (int j = 0; j < 6; ++j, ++idx) {
      ok = ok && same(P[idx].grad, grads.data() + off);
      off += static_cast<std::size_t>(P[idx].grad.elems());
    }
  {
    std::vector<T> v(static_cast<std::size_t>(c_out));
    to_flat(dhg, v.data());
    ok = ok && same(P[hb].grad, v.data());
    to_flat(dhb, v.data());
    ok = ok && same(P[hb + 1].grad, v.data());
  }
  if (!ok) throw VerifyError("block harness disagrees with GraphPlan::step_trace");
}

DenseNetConfig model_cfg(int nblocks, const int* blocks, int k, int bottleneck,
                         double compression, int classes, int c0) {
  return build_config(std::vector<int>(blocks, blocks + nblocks), k,
                      bottleneck != 0, compression,
                      ActivationOrder::PreActivation, classes, c0);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

#define DEFINE_HARNESS(SUF, T)                                                 \
  int ref_block_harness_##SUF(std::int64_t n, std::int64_t h, std::int64_t w,  \
                              std::int64_t c0, std::int64_t m, std::int64_t k, \
                              std::int64_t bk, const T* params, const T* x_in, \
                              T* running, int update_running, T* feats,        \
                              T* z, T* stats, T* acc, T* grads) {              \
    return guarded([&] {                                                       \
      block_harness<T>(n, h, w, c0, m, k, bk, params, x_in, running,           \
                       update_running, feats, z, stats, acc, grads);           \
    });                                                                        \
  }                                                                            \
  int ref_check_block_harness_##SUF(int m, int k, int c0, int n, int h, int w, \
                                    std::uint64_t seed) {                      \
    return guarded([&] { check_block_harness<T>(m, k, c0, n, h, w, seed); });  \
  }
DEFINE_HARNESS(f32, float)
DEFINE_HARNESS(f64, double)

// Parameters exactly as GraphPlan<T>::build draws them (He-normal, BN 1/0),
// for a model config; writes the flat block-layer params of block `b`.
int ref_block_params_f32(int nblocks, const int* blocks, int k, int bottleneck,
                         double compression, int classes, int c0, int in_c,
                         int in_h, int in_w, std::int64_t batch,
                         std::uint64_t seed, int b, float* out) {
  return guarded([&] {
    const DenseNetConfig cfg = model_cfg(nblocks, blocks, k, bottleneck,
                                         compression, classes, c0);
    GraphPlan<float> plan = GraphPlan<float>::build(
        cfg, ExecutionStrategy::SharedAll, Shape4{batch, in_c, in_h, in_w}, seed);
    const std::string pre = "b" + std::to_string(b) + ".l";
    std::size_t off = 0;
    for (const auto& p : plan.params()) {
      if (p.name.rfind(pre, 0) != 0) continue;
      to_flat(p.value, out + off);
      off += static_cast<std::size_t>(p.value.elems());
    }
  });
}

// Every parameter of a freshly built GraphPlan in registration order
// (stem.w, b*.l*, t*.bn/conv, head.bn, head.linear) and the reference's
// synthetic input Rng(seed+99).normal() (NCHW).  Either pointer may be null.
int ref_model_params_f32(int nblocks, const int* blocks, int k, int bottleneck,
                         double compression, int classes, int c0, int in_c,
                         int in_h, int in_w, std::int64_t batch,
                         std::uint64_t seed, float* params, float* input) {
  return guarded([&] {
    const DenseNetConfig cfg = model_cfg(nblocks, blocks, k, bottleneck,
                                         compression, classes, c0);
    const Shape4 in{batch, in_c, in_h, in_w};
    if (params != nullptr) {
      GraphPlan<float> plan =
          GraphPlan<float>::build(cfg, ExecutionStrategy::SharedAll, in, seed);
      std::size_t off = 0;
      for (const auto& p : plan.params()) {
        to_flat(p.value, params + off);
        off += static_cast<std::size_t>(p.value.elems());
      }
    }
    if (input != nullptr) {
      MemoryTracker data_tr;
      to_flat(make_input<float>(in, seed + 99, data_tr), input);
    }
  });
}

// One reference training step (GraphPlan::step_trace, SharedAll) on the
// reference's synthetic input Rng(seed+99).normal() / labels i % classes.
// Writes the loss, the step wall time in seconds, and (when `grads` is not
// null) all parameter gradients concatenated in registration order.
int ref_model_step_f32(int nblocks, const int* blocks, int k, int bottleneck,
                       double compression, int classes, int c0, int in_c,
                       int in_h, int in_w, std::int64_t batch,
                       std::uint64_t seed, int steps, double* loss,
                       double* best_seconds, float* grads) {
  return guarded([&] {
    const DenseNetConfig cfg = model_cfg(nblocks, blocks, k, bottleneck,
                                         compression, classes, c0);
    const Shape4 in{batch, in_c, in_h, in_w};
    MemoryTracker data_tr;
    Tensor<float> input = make_input<float>(in, seed + 99, data_tr);
    const std::vector<int> labels = make_labels(static_cast<int>(batch), classes);
    GraphPlan<float> plan =
        GraphPlan<float>::build(cfg, ExecutionStrategy::SharedAll, in, seed);
    double best = 1e300;
    for (int s = 0; s < steps; ++s) {
      const auto t0 = std::chrono::steady_clock::now();
      const StepResult<float> r = plan.step_trace(input, labels);
      const auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
      *loss = r.loss;
    }
    *best_seconds = best;
    if (grads != nullptr) {
      std::size_t off = 0;
      for (const auto& p : plan.params()) {
        to_flat(p.grad, grads + off);
        off += static_cast<std::size_t>(p.grad.elems());
      }
    }
  });
}

}  // extern "C"

// ---- one training step with running statistics (F10) and the ImageNet stem --------
//
// ref_model_train_step_f32 runs the reference's PUBLIC GraphPlan<float>
// forward(Train) / compute_loss / backward (graph.hpp:726-826, 1065-1183) and
// returns the loss, every parameter gradient and the BN running statistics
// after the step.  GraphPlan keeps its BN states private and checkpoints omit
// them, so the running statistics are derived from the public
// StepState statistics with the reference's own momentum expression
// (ops.hpp:185-194): r = (1 - 0.1f) * r0 + 0.1f * stat, r0 = (0, 1).
//
// stem 0: the reference network as is.  stem 1: the ImageNet stem (conv
// 7x7/2 pad 3 -> BN -> ReLU -> max-pool 3x3/2 pad 1), which the reference does
// not have, composed from the reference's public ops:: (conv2d_forward /
// conv2d_backward with stride 2, batchnorm_forward / batchnorm_backward,
// relu_inplace / relu_backward_inplace) plus a restated max-pool (first
// maximum in (ky, kx) order wins; its backward scatters in (n, c, oy, ox)
// order).  The rest of the network is the unmodified GraphPlan run on the
// stem output with an identity 3x3 stem (centre tap 1: conv2d_forward then
// returns its input exactly) under the Naive strategy — bitwise equal to
// SharedAll (t/graph_test.cpp:99-111) — whose StepState.retained keeps the
// block-0 gradient accumulator, the gradient w.r.t. the stem output.
//
// Flat layouts are libdpb's (include/dpb.h dpb_model_*): params / grads in
// registration order with the stem first; running = (stem 1: stem mean, var)
// then per block its per-layer (mean_a, var_a, mean_b, var_b), then the
// transition / head (mean, var).  params may be null (GraphPlan::build init,
// stem 0 only); x may be null (Rng(seed + 99).normal(), NCHW).
namespace {

template <typename T>
T run_update(T r0, T stat) {  // ops.hpp:190-193
  const T momentum = static_cast<T>(0.1);
  return (T(1) - momentum) * r0 + momentum * stat;
}

template <typename T>
void put_running(const ops::BatchStats<T>& st, T*& out) {
  for (T v : st.mean) *out++ = run_update(T(0), v);
  for (T v : st.var) *out++ = run_update(T(1), v);
}

// float host data -> a Tensor<T> (exact for T = double)
template <typename T>
Tensor<T> from_float(const float* src, const Shape4& s, MemoryTracker& tr) {
  Tensor<T> t = Tensor<T>::alloc(s, ArenaTag::Scratch, tr);
  for (std::int64_t i = 0; i < s.elems(); ++i) t.data()[i] = static_cast<T>(src[i]);
  return t;
}

template <typename T>
struct MaxPool3 {  // 3x3 stride 2 pad 1 max-pool, restated (not in the reference)
  std::vector<int> arg;  // per output: input flat index of the first maximum
  Shape4 os;
  void forward(const Tensor<T>& x, Tensor<T>& y) {
    const Shape4& s = x.shape();
    os = y.shape();
    arg.assign(static_cast<std::size_t>(os.elems()), -1);
    std::size_t o = 0;
    for (std::int64_t i = 0; i < s.n; ++i)
      for (std::int64_t c = 0; c < s.c; ++c)
        for (std::int64_t oy = 0; oy < os.h; ++oy)
          for (std::int64_t ox = 0; ox < os.w; ++ox, ++o) {
            T best = 0;
            int bi = -1;
            for (std::int64_t ky = 0; ky < 3; ++ky) {
              const std::int64_t iy = 2 * oy - 1 + ky;
              if (iy < 0 || iy >= s.h) continue;
              for (std::int64_t kx = 0; kx < 3; ++kx) {
                const std::int64_t ix = 2 * ox - 1 + kx;
                if (ix < 0 || ix >= s.w) continue;
                const T v = x.at(i, c, iy, ix);
                if (bi < 0 || v > best) {
                  best = v;
                  bi = static_cast<int>(((i * s.c + c) * s.h + iy) * s.w + ix);
                }
              }
            }
            y.at(i, c, oy, ox) = best;
            arg[o] = bi;
          }
  }
  void backward(const Tensor<T>& gy, Tensor<T>& gx) {
    gx.fill(T(0));
    std::size_t o = 0;
    for (std::int64_t i = 0; i < os.n; ++i)
      for (std::int64_t c = 0; c < os.c; ++c)
        for (std::int64_t oy = 0; oy < os.h; ++oy)
          for (std::int64_t ox = 0; ox < os.w; ++ox, ++o) gx.data()[arg[o]] += gy.at(i, c, oy, ox);
  }
};

template <typename T>
void model_train_step(int nblocks, const int* blocks, int k, double compression, int classes, int c0, int stem,
                      int in_c, int in_h, int in_w, std::int64_t batch, std::uint64_t seed, const float* params,
                      const float* x_in, double* loss, T* grads, T* running) {
  const int kk = stem == 1 ? 7 : 3;
  MemoryTracker tr;
  const Shape4 in{batch, in_c, in_h, in_w};
  // the float synthetic input Rng(seed+99) (make_input<float>), exact in T
  Tensor<T> input;
  if (x_in) {
    input = from_float<T>(x_in, in, tr);
  } else {
    Tensor<float> xf = make_input<float>(in, seed + 99, tr);
    input = from_float<T>(xf.data(), in, tr);
  }
  const std::vector<int> labels = make_labels(static_cast<int>(batch), classes);

  // ---- stem 1 forward (reference ops + restated max-pool) ----
  ops::ConvParams<T> sconv;
  ops::BatchNormState<T> sbn;
  ops::BatchStats<T> sstats;
  Tensor<T> sy, sact, spool;
  MaxPool3<T> pool;
  const std::int64_t swn = static_cast<std::int64_t>(c0) * in_c * kk * kk;
  if (stem == 1) {
    if (params == nullptr) throw ConfigError("the ImageNet stem needs explicit parameters");
    sconv.weights = from_float<T>(params, Shape4{c0, in_c, 7, 7}, tr);
    sconv.stride = 2;
    sconv.padding = 3;
    const std::vector<T> r0(static_cast<std::size_t>(c0), T(0)), r1(static_cast<std::size_t>(c0), T(1));
    const std::vector<T> gm(params + swn, params + swn + c0), bt(params + swn + c0, params + swn + 2 * c0);
    sbn = make_bn(gm.data(), bt.data(), r0.data(), r1.data(), c0, tr);
    const Shape4 ys = ops::conv2d_out_shape(in, sconv);
    sy = Tensor<T>::alloc(ys, ArenaTag::Scratch, tr);
    ops::conv2d_forward(input, sconv, sy);
    sact = Tensor<T>::alloc(ys, ArenaTag::Scratch, tr);
    sstats = ops::batchnorm_forward(sy, sbn, ops::BnMode::Train, sact, true);
    ops::relu_inplace(sact);
    const Shape4 ps{batch, c0, (ys.h + 2 - 3) / 2 + 1, (ys.w + 2 - 3) / 2 + 1};
    spool = Tensor<T>::alloc(ps, ArenaTag::Scratch, tr);
    pool.forward(sact, spool);
  }
  const std::int64_t soff = stem == 1 ? swn + 2 * c0 : swn;  // params after the stem

  // ---- the reference network ----
  const DenseNetConfig cfg = model_cfg(nblocks, blocks, k, 1, compression, classes, c0);
  const Shape4 gin = stem == 1 ? spool.shape() : in;
  GraphPlan<T> plan =
      GraphPlan<T>::build(cfg, stem == 1 ? ExecutionStrategy::Naive : ExecutionStrategy::SharedAll, gin, seed);
  {
    std::size_t off = 0;
    for (auto& p : plan.params()) {
      const std::int64_t n = p.value.elems();
      if (p.name == "stem.conv.w") {
        if (stem == 1) {  // identity 3x3: out[o] = in[o]
          p.value.fill(T(0));
          for (std::int64_t o = 0; o < c0; ++o) p.value.at(o, o, 1, 1) = T(1);
        } else if (params) {
          for (std::int64_t i = 0; i < n; ++i) p.value.data()[i] = static_cast<T>(params[i]);
        }
        off = static_cast<std::size_t>(soff);
        continue;
      }
      if (params)
        for (std::int64_t i = 0; i < n; ++i) p.value.data()[i] = static_cast<T>(params[off + static_cast<std::size_t>(i)]);
      off += static_cast<std::size_t>(n);
    }
  }
  StepState<T> state = plan.forward(stem == 1 ? spool : input, ops::BnMode::Train);
  *loss = plan.compute_loss(state, labels);
  plan.backward(state);

  // gradients (registration order), the stem's from the composition below
  {
    std::size_t off = 0;
    for (const auto& p : plan.params()) {
      const std::int64_t n = p.grad.elems();
      if (p.name == "stem.conv.w") {
        if (stem == 0) to_flat(p.grad, grads);
        off = static_cast<std::size_t>(soff);
        continue;
      }
      to_flat(p.grad, grads + off);
      off += static_cast<std::size_t>(n);
    }
  }
  // running statistics (F10)
  T* r = running;
  if (stem == 1) put_running(sstats, r);
  for (std::size_t b = 0; b < state.blocks.size(); ++b) {
    for (const auto& ls : state.blocks[b].layers) {
      put_running(ls.stats_a, r);
      put_running(ls.stats_b, r);
    }
    put_running(b + 1 < state.blocks.size() ? state.trans[b].stats : state.head.stats, r);
  }

  // ---- stem 1 backward ----
  if (stem == 1) {
    const Shape4 ps = spool.shape();
    const std::int64_t C0out = c0 + static_cast<std::int64_t>(blocks[0]) * k;
    // Naive backward retains, in order, ..., the block-0 accumulator (acquired by
    // transition 0 or the head), then block 0's four transients per layer
    // (backward_layer, graph.hpp:905-935); the stem's wgrad acquires nothing.
    const std::size_t nr = state.retained.size(), after = 4 * static_cast<std::size_t>(blocks[0]);
    if (nr < after + 1) throw AccountingError("block-0 accumulator not retained");
    const Tensor<T>* acc0 = &state.retained[nr - after - 1];
    if (acc0->shape() != Shape4{ps.n, C0out, ps.h, ps.w}) throw AccountingError("block-0 accumulator shape");
    Tensor<T> gpool = Tensor<T>::alloc(ps, ArenaTag::Scratch, tr);
    for (std::int64_t i = 0; i < ps.n; ++i)
      for (std::int64_t c = 0; c < c0; ++c)
        for (std::int64_t y = 0; y < ps.h; ++y)
          for (std::int64_t x = 0; x < ps.w; ++x) gpool.at(i, c, y, x) = acc0->at(i, c, y, x);
    Tensor<T> ga = Tensor<T>::alloc(sy.shape(), ArenaTag::Scratch, tr);
    pool.backward(gpool, ga);
    ops::relu_backward_inplace(ga, sact);
    Tensor<T> gy = Tensor<T>::alloc(sy.shape(), ArenaTag::Scratch, tr);
    Tensor<T> dg = Tensor<T>::alloc(Shape4{1, c0, 1, 1}, ArenaTag::Scratch, tr);
    Tensor<T> db = Tensor<T>::alloc(Shape4{1, c0, 1, 1}, ArenaTag::Scratch, tr);
    ops::batchnorm_backward(ga, sy, sbn, sstats, gy, dg, db);
    Tensor<T> dw = Tensor<T>::alloc(sconv.weights.shape(), ArenaTag::Scratch, tr);
    ops::conv2d_backward(gy, input, sconv, static_cast<Tensor<T>*>(nullptr), dw);
    to_flat(dw, grads);
    to_flat(dg, grads + swn);
    to_flat(db, grads + swn + c0);
  }
}

}  // namespace

// OpTrace of one GraphPlan<double> step (alloctrace.hpp:132-201) of the
// single-block network blocks={m} (single_block_cfg, 4 classes), strategy
// 0 naive / 1 shared-gradient / 2 shared-all: per-node {forward, backward,
// recompute} counts and per-OpKind FLOPs {forward, backward, recompute}.
extern "C" int ref_single_block_trace(int m, int k, int c0, int n, int h, int w, std::uint64_t seed, int strategy,
                                      int32_t* counts, int max_nodes, double* flops, int* nodes) {
  return guarded([&] {
    const DenseNetConfig cfg = single_block_cfg(m, k, c0, 4);
    const Shape4 in{n, 3, h, w};
    MemoryTracker data_tr;
    Tensor<double> input = make_input<double>(in, seed + 99, data_tr);
    GraphPlan<double> plan = GraphPlan<double>::build(cfg, static_cast<ExecutionStrategy>(strategy), in, seed);
    const StepResult<double> r = plan.step_trace(input, make_labels(n, 4));
    *nodes = static_cast<int>(r.trace.node_count());
    for (int i = 0; i < *nodes && i < max_nodes; ++i) {
      const OpTrace::NodeCounts& c = r.trace.node(i);
      counts[3 * i] = c.forward;
      counts[3 * i + 1] = c.backward;
      counts[3 * i + 2] = c.recompute;
    }
    for (int kk = 0; kk < kOpKindCount; ++kk) {
      flops[kk] = r.trace.forward_flops(static_cast<OpKind>(kk));
      flops[7 + kk] = r.trace.backward_flops(static_cast<OpKind>(kk));
      flops[14 + kk] = r.trace.recompute_flops(static_cast<OpKind>(kk));
    }
  });
}

#define DEFINE_TRAIN_STEP(SUF, T)                                                                               \
  extern "C" int ref_model_train_step_##SUF(int nblocks, const int* blocks, int k, double compression,         \
                                            int classes, int c0, int stem, int in_c, int in_h, int in_w,        \
                                            std::int64_t batch, std::uint64_t seed, const float* params,        \
                                            const float* x, double* loss, T* grads, T* running) {               \
    return guarded([&] {                                                                                        \
      model_train_step<T>(nblocks, blocks, k, compression, classes, c0, stem, in_c, in_h, in_w, batch, seed,    \
                          params, x, loss, grads, running);                                                    \
    });                                                                                                         \
  }
DEFINE_TRAIN_STEP(f32, float)
DEFINE_TRAIN_STEP(f64, double)

extern "C" {

// The reference's sgd_step (train.hpp:43-70) over one flat parameter of n
// elements: params / velocity updated in place from grads.
int ref_sgd_step_f32(float* params, const float* grads, float* velocity, std::int64_t n, double lr,
                     double momentum, double weight_decay, int nesterov) {
  return guarded([&] {
    MemoryTracker tr;
    std::vector<ParamEntry<float>> reg;
    reg.push_back({"p", from_flat(params, Shape4{1, n, 1, 1}, tr), from_flat(grads, Shape4{1, n, 1, 1}, tr)});
    OptimizerState<float> opt = OptimizerState<float>::create(reg);
    std::memcpy(opt.velocity[0].data(), velocity, sizeof(float) * static_cast<std::size_t>(n));
    opt.momentum = momentum;
    opt.weight_decay = weight_decay;
    opt.nesterov = nesterov != 0;
    sgd_step(reg, opt, lr);
    to_flat(reg[0].value, params);
    to_flat(opt.velocity[0], velocity);
  });
}

// The reference's save_training_checkpoint (train.hpp:157-162) of a fresh
// GraphPlan (seed) with velocities v_i = 0.5 * p_i.
int ref_save_training_checkpoint(int nblocks, const int* blocks, int k, int bottleneck, double compression,
                                 int classes, int c0, int in_c, int in_h, int in_w, std::int64_t batch,
                                 std::uint64_t seed, const char* path, int epoch) {
  return guarded([&] {
    const DenseNetConfig cfg = model_cfg(nblocks, blocks, k, bottleneck, compression, classes, c0);
    GraphPlan<float> plan =
        GraphPlan<float>::build(cfg, ExecutionStrategy::SharedAll, Shape4{batch, in_c, in_h, in_w}, seed);
    OptimizerState<float> opt = OptimizerState<float>::create(plan.params());
    for (std::size_t i = 0; i < opt.velocity.size(); ++i) {
      const Tensor<float>& p = plan.params()[i].value;
      for (std::int64_t j = 0; j < p.elems(); ++j) opt.velocity[i].data()[j] = 0.5f * p.data()[j];
    }
    save_training_checkpoint(path, plan, opt, epoch);
  });
}

// config_to_text(preset_config(name)) (densenet.hpp:89-115, 279-297) into out[cap].
int ref_preset_text(const char* name, char* out, int cap) {
  return guarded([&] {
    const std::string t = config_to_text(preset_config(name));
    std::snprintf(out, static_cast<std::size_t>(cap), "%s", t.c_str());
  });
}

// config_to_text(config_from_key_values(parse_key_values(text))): the round trip.
int ref_config_roundtrip(const char* text, char* out, int cap) {
  return guarded([&] {
    std::istringstream in(text);
    const std::string t = config_to_text(config_from_key_values(parse_key_values(in)));
    std::snprintf(out, static_cast<std::size_t>(cap), "%s", t.c_str());
  });
}

// config_from_key_values(parse_key_values(text)) (densenet.hpp:300-370): the
// parsed configuration's fields, or the reference's error (ref_last_error).
int ref_parse_config(const char* text, int* blocks, int cap, int* nblocks, int* k, int* bottleneck,
                     double* compression, int* c0, int* post, int* classes) {
  return guarded([&] {
    std::istringstream in(text);
    const DenseNetConfig cfg = config_from_key_values(parse_key_values(in));
    *nblocks = static_cast<int>(cfg.block_sizes.size());
    for (int i = 0; i < *nblocks && i < cap; ++i) blocks[i] = cfg.block_sizes[i];
    *k = cfg.growth_rate;
    *bottleneck = cfg.bottleneck ? 1 : 0;
    *compression = cfg.compression;
    *c0 = cfg.initial_channels;
    *post = cfg.activation_order == ActivationOrder::PostActivation ? 1 : 0;
    *classes = cfg.num_classes;
  });
}

// lr_at (schedule.hpp:46-62): kind 0 = Step (milestones, factor), 1 = Cosine (floor).
int ref_lr_at(int kind, double base_lr, int total_epochs, const int* milestones, int nmilestones,
              double factor, double floor, int epoch, double* out) {
  return guarded([&] {
    LrSchedule s;
    s.kind = kind == 1 ? ScheduleKind::Cosine : ScheduleKind::Step;
    s.base_lr = base_lr;
    s.total_epochs = total_epochs;
    s.milestones.assign(milestones, milestones + nmilestones);
    s.factor = factor;
    s.floor = floor;
    *out = lr_at(s, epoch);
  });
}

// Rng(seed).normal() x count (dp/rng.hpp:36-49) and raw next_u64 draws.
void ref_rng_normal(std::uint64_t seed, std::int64_t count, double* out) {
  Rng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.normal();
}
void ref_rng_u64(std::uint64_t seed, std::int64_t count, std::uint64_t* out) {
  Rng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

std::int64_t ref_count_parameters(int nblocks, const int* blocks, int k,
                                  int bottleneck, double compression,
                                  int classes, int c0, int in_c) {
  std::int64_t r = -1;
  guarded([&] {
    r = count_parameters(
        model_cfg(nblocks, blocks, k, bottleneck, compression, classes, c0), in_c);
  });
  return r;
}

// predict_peak_elements (dp/peak_model.hpp:37-158): out[6] per-arena elems.
int ref_predict_peak_elements(int nblocks, const int* blocks, int k,
                              int bottleneck, double compression, int classes,
                              int c0, int strategy, std::int64_t batch,
                              int in_c, int in_h, int in_w, std::int64_t* out) {
  return guarded([&] {
    const PeakPrediction p = predict_peak_elements(
        model_cfg(nblocks, blocks, k, bottleneck, compression, classes, c0),
        static_cast<ExecutionStrategy>(strategy), batch, in_c, in_h, in_w);
    for (int i = 0; i < kArenaCount; ++i) out[i] = p.elems[static_cast<std::size_t>(i)];
  });
}

}  // extern "C"
