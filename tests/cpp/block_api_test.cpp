// C++ host API test (include/denseplan_b200/block.hpp), written like the
// reference's own doctest suites (t/graph_test.cpp, t/alloctrace_test.cpp).
// `block_api_test --host` runs the host-only checks (no GPU needed).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "denseplan_b200/block.hpp"

using namespace denseplan_b200;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("[FAIL] %s:%d %s\n", __FILE__, __LINE__, #cond);         \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <typename E, typename F>
static bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void host_checks() {
  // t/densenet_test.cpp:214-231 and BASELINE's 33M / 73M models
  CHECK(count_parameters({26, 26, 26}, 12, true, 0.5, 10, 24) == 1739002);
  CHECK(count_parameters({6, 12, 64, 48}, 32, true, 0.5, 1000, 64) == 33329896);
  CHECK(count_parameters({6, 12, 64, 48}, 48, true, 0.5, 1000, 96) == 72674920);
  // Shape4 overflow guard (tensor.hpp:34-36)
  CHECK(throws_as<SizeOverflowError>([] { Shape4{1LL << 40, 1LL << 20, 1, 1}.elems(); }));
  CHECK(throws_as<ShapeError>([] { Shape4{0, 1, 1, 1}.elems(); }));
  // arena plan: O(m) features, no Shared1/Shared2 pools
  BlockConfig cfg{16, 32, 32, 24, 12, 12, 48, Precision::BF16, Layout::NCHW};
  const ArenaPlan a = plan_arena(cfg);
  CHECK(a.bytes(ArenaTag::Shared1) == 0 && a.bytes(ArenaTag::Shared2) == 0);
  CHECK(a.raw.feat_bytes == 16LL * 32 * 32 * 168 * 4);
  CHECK(a.raw.z_bytes == 12LL * 16 * 32 * 32 * 48 * 4);
  CHECK(a.total() >= a.bytes(ArenaTag::FeatureOwned) + a.bytes(ArenaTag::SharedGrad));
  BlockConfig bad = cfg;
  bad.c0 = 0;
  CHECK(throws_as<ShapeError>([&] { plan_arena(bad); }));
  bad = cfg;
  bad.layout = static_cast<Layout>(9);
  CHECK(throws_as<ConfigError>([&] { plan_arena(bad); }));
}

static void device_checks() {
  BlockConfig cfg{2, 8, 8, 16, 3, 8, 32, Precision::FP32, Layout::NCHW};
  BlockPlan plan = BlockPlan::build(cfg);
  const std::int64_t P = plan.param_elems(), S = plan.stat_elems();
  const std::int64_t xin = cfg.n * cfg.c0 * cfg.h * cfg.w;
  const std::int64_t acc_n = cfg.n * cfg.c_out() * cfg.h * cfg.w;
  std::mt19937_64 eng(7);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> hp(P), hx(xin), hr(S, 0.f), hacc(acc_n, 0.f), hg(P, 7.f);
  for (auto& v : hp) v = 0.2f * nd(eng);
  for (auto& v : hx) v = nd(eng);
  // running mean 0 / var 1 (graph.hpp:358-360): var slots per layer
  std::int64_t o = 0;
  for (int l = 0; l < cfg.layers; ++l) {
    const int c = cfg.c_in(l), bk = 4 * cfg.growth_rate;
    for (int i = 0; i < c; ++i) hr[o + c + i] = 1.f;
    for (int i = 0; i < bk; ++i) hr[o + 2 * c + bk + i] = 1.f;
    o += 2 * c + 2 * bk;
  }
  float *dp, *dx, *dr, *dacc, *dg;
  cudaMalloc(&dp, P * 4);
  cudaMalloc(&dx, xin * 4);
  cudaMalloc(&dr, S * 4);
  cudaMalloc(&dacc, acc_n * 4);
  cudaMalloc(&dg, P * 4);
  cudaMemcpy(dp, hp.data(), P * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, hx.data(), xin * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, hr.data(), S * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dacc, hacc.data(), acc_n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dg, hg.data(), P * 4, cudaMemcpyHostToDevice);

  // backward before a train-mode forward: ProtocolError (graph.hpp:1067-1070)
  CHECK(throws_as<ProtocolError>([&] { plan.backward(dp, dacc, dg); }));
  plan.forward(dx, dp, dr);
  // zero upstream gradient -> zero parameter gradients (t/graph_test.cpp:164-185)
  plan.backward(dp, dacc, dg);
  plan.sync();
  cudaMemcpy(hg.data(), dg, P * 4, cudaMemcpyDeviceToHost);
  bool all_zero = true;
  for (float v : hg) all_zero = all_zero && v == 0.f;
  CHECK(all_zero);
  // running stats moved by the momentum rule; frozen stats do not move
  std::vector<float> r1(S), r2(S);
  cudaMemcpy(r1.data(), dr, S * 4, cudaMemcpyDeviceToHost);
  CHECK(std::memcmp(r1.data(), hr.data(), S * 4) != 0);
  plan.set_freeze_running_stats(true);
  plan.forward(dx, dp, dr);
  plan.sync();
  cudaMemcpy(r2.data(), dr, S * 4, cudaMemcpyDeviceToHost);
  CHECK(std::memcmp(r1.data(), r2.data(), S * 4) == 0);
  // block output: channels [0, c0) are the block input (zero-copy concat)
  std::vector<float> feats(acc_n);
  float* dfeats;
  cudaMalloc(&dfeats, acc_n * 4);
  plan.read_feats(dfeats);
  plan.sync();
  cudaMemcpy(feats.data(), dfeats, acc_n * 4, cudaMemcpyDeviceToHost);
  bool copied = true;
  const std::int64_t hw = cfg.h * cfg.w;
  for (std::int64_t i = 0; i < cfg.n; ++i)
    for (std::int64_t c = 0; c < cfg.c0; ++c)
      for (std::int64_t p = 0; p < hw; ++p)
        copied = copied && feats[(i * cfg.c_out() + c) * hw + p] == hx[(i * cfg.c0 + c) * hw + p];
  CHECK(copied);
  // degenerate batch: n*h*w < 2 (ops.hpp:180-183)
  BlockConfig tiny{1, 1, 1, 4, 1, 2, 8, Precision::FP32, Layout::NCHW};
  BlockPlan t = BlockPlan::build(tiny);
  CHECK(throws_as<DegenerateBatchError>([&] { t.forward(dx, dp, dr); }));
  cudaFree(dp);
  cudaFree(dx);
  cudaFree(dr);
  cudaFree(dacc);
  cudaFree(dg);
  cudaFree(dfeats);
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::string(argv[1]) == "--host";
  host_checks();
  if (!host_only) device_checks();
  std::printf("%s: %d failure(s)\n", failures ? "[FAIL]" : "[PASS]", failures);
  return failures ? 1 : 0;
}
