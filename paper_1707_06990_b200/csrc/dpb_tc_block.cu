// Launchers of the tcgen05 convolution ops (dpb_tc_ops.cuh) for one layer of
// the block; called by dpb_block.cu when the block runs the tensor-core path
// (DPB_BF16).
#include <cuda_runtime.h>

#include <algorithm>

#include "dpb_internal.h"
#include "dpb_tc_ops.cuh"

namespace dpb {

using tc::TcArgs;

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

bool tc_supported(const dpb_block_desc& d) {
  // chunks of 8 channels never straddle a 3x3 tap; N tiles the engine has
  return d.bk % 8 == 0 && d.bk <= 256 && d.k <= 64;
}

template <class Op>
static void launch(Block* b, const Op& op, dim3 grid, size_t aux) {
  static int max_dyn = -1;
  if (max_dyn < 0) {
    // opt in to the full 227 KB minus the kernel's static shared memory
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, tc::tc_gemm_kernel<Op>);
    max_dyn = 227 * 1024 - static_cast<int>(fa.sharedSizeBytes);
    cudaFuncSetAttribute(tc::tc_gemm_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         max_dyn);
  }
  const size_t smem = tc::stage_bytes<Op>() + aux;
  tc::tc_gemm_kernel<Op><<<grid, tc::kThreads, smem, b->stream>>>(op);
}

// N tile for an N of `n` channels from the instantiated set.
static int pick_bn(int n) {
  const int r = round_up(n, 16);
  if (r <= 16) return 16;
  if (r <= 32) return 32;
  if (r <= 48) return 48;
  if (r <= 64) return 64;
  if (r <= 128) return 128;
  if (r <= 192) return 192;
  return 256;
}

template <template <int> class Op>
static void launch_bn(Block* b, int bn, const TcArgs& t, dim3 grid, size_t aux) {
  switch (bn) {
    case 16: launch(b, Op<16>{t}, grid, aux); break;
    case 32: launch(b, Op<32>{t}, grid, aux); break;
    case 48: launch(b, Op<48>{t}, grid, aux); break;
    case 64: launch(b, Op<64>{t}, grid, aux); break;
    case 128: launch(b, Op<128>{t}, grid, aux); break;
    case 192: launch(b, Op<192>{t}, grid, aux); break;
    default: launch(b, Op<256>{t}, grid, aux); break;
  }
}

template <template <int> class Op>
static void launch_small(Block* b, int bn, const TcArgs& t, dim3 grid, size_t aux) {
  switch (bn) {
    case 16: launch(b, Op<16>{t}, grid, aux); break;
    case 32: launch(b, Op<32>{t}, grid, aux); break;
    case 48: launch(b, Op<48>{t}, grid, aux); break;
    default: launch(b, Op<64>{t}, grid, aux); break;
  }
}

static TcArgs make_args(const LayerArgs<float>& a) {
  TcArgs t{};
  t.a = a;
  t.kp = round_up(a.k, 8);
  t.vec = (a.C % 4 == 0) && (a.c % 4 == 0);
  return t;
}

static unsigned mtiles(int64_t rows) { return static_cast<unsigned>((rows + tc::kBM - 1) / tc::kBM); }

void tc_conv1x1_fwd(Block* b, const LayerArgs<float>& a) {
  const TcArgs t = make_args(a);
  launch_bn<tc::Tc1x1Fwd>(b, pick_bn(a.bk), t, dim3(mtiles(a.M)), sizeof(BnFwd) * a.c);
}

void tc_conv3x3_fwd(Block* b, const LayerArgs<float>& a) {
  const TcArgs t = make_args(a);
  launch_small<tc::Tc3x3Fwd>(b, pick_bn(a.k), t, dim3(mtiles(a.M)),
                             sizeof(BnFwd) * a.bk + sizeof(int) * tc::kBM);
}

void tc_conv3x3_dgrad(Block* b, const LayerArgs<float>& a) {
  const TcArgs t = make_args(a);
  launch_bn<tc::Tc3x3Dgrad>(b, pick_bn(a.bk), t, dim3(mtiles(a.M)),
                            sizeof(BnFwd) * a.bk + sizeof(int) * tc::kBM);
}

void tc_conv1x1_dgrad(Block* b, const LayerArgs<float>& a) {
  const TcArgs t = make_args(a);
  const int bn = a.c <= 64 ? 64 : 128;
  const size_t aux = (sizeof(BnBwd) * a.bk + 15) / 16 * 16 + sizeof(BnFwd) * bn;
  const dim3 grid(mtiles(a.M), static_cast<unsigned>((a.c + bn - 1) / bn));
  if (bn == 64) launch(b, tc::Tc1x1Dgrad<64>{t}, grid, aux);
  else launch(b, tc::Tc1x1Dgrad<128>{t}, grid, aux);
}

// Split-K over pixels for the weight gradients: ~2 waves of 148 SMs, chunks
// a multiple of the K block.
int64_t tc_wgrad_chunk(int64_t M, int64_t tiles) {
  int64_t splits = std::max<int64_t>(1, 296 / std::max<int64_t>(1, tiles));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, M / 512));
  int64_t chunk = (M + splits - 1) / splits;
  return (chunk + tc::kBK - 1) / tc::kBK * tc::kBK;
}

int tc_conv1x1_wgrad(Block* b, LayerArgs<float> a) {
  const int64_t tiles = mtiles(a.c);
  a.kchunk = tc_wgrad_chunk(a.M, tiles);
  const int splits = static_cast<int>((a.M + a.kchunk - 1) / a.kchunk);
  const TcArgs t = make_args(a);
  const size_t aux = (sizeof(BnBwd) * a.bk + 15) / 16 * 16 + sizeof(BnFwd) * tc::kBM;
  launch_bn<tc::Tc1x1Wgrad>(b, pick_bn(a.bk), t, dim3(mtiles(a.c), 1, splits), aux);
  return splits;
}

int tc_conv3x3_wgrad(Block* b, LayerArgs<float> a) {
  const int64_t tiles = mtiles(9LL * a.bk);
  a.kchunk = tc_wgrad_chunk(a.M, tiles);
  const int splits = static_cast<int>((a.M + a.kchunk - 1) / a.kchunk);
  const TcArgs t = make_args(a);
  launch_small<tc::Tc3x3Wgrad>(b, pick_bn(a.k), t, dim3(mtiles(9LL * a.bk), 1, splits),
                               sizeof(BnFwd) * a.bk);
  return splits;
}

}  // namespace dpb
