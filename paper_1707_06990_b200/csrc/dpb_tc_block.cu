// Launchers of the tcgen05 convolution ops (dpb_tc_ops.cuh) for one layer of
// the block; called by dpb_block.cu when the block runs the tensor-core path
// (DPB_BF16).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "dpb_internal.h"
#include "dpb_launch.h"
#include "dpb_tc_halo.cuh"
#include "dpb_tc_ops.cuh"

namespace dpb {

using tc::TcArgs;

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

bool tc_supported(const dpb_block_desc& d) {
  // chunks of 8 channels never straddle a 3x3 tap; N tiles the engine has
  return d.bk % 8 == 0 && d.bk <= 256 && d.k <= 64;
}

template <class Op>
static void launch_tc(Block* b, const Op& op, dim3 grid, size_t aux) {
  const size_t smem = tc::stage_bytes<Op>() + aux;
  launch(tc::tc_gemm_kernel<Op>, grid, tc::kThreads, smem, b->stream, op);
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
    case 16: launch_tc(b, Op<16>{t}, grid, aux); break;
    case 32: launch_tc(b, Op<32>{t}, grid, aux); break;
    case 48: launch_tc(b, Op<48>{t}, grid, aux); break;
    case 64: launch_tc(b, Op<64>{t}, grid, aux); break;
    case 128: launch_tc(b, Op<128>{t}, grid, aux); break;
    case 192: launch_tc(b, Op<192>{t}, grid, aux); break;
    default: launch_tc(b, Op<256>{t}, grid, aux); break;
  }
}

template <template <int> class Op>
static void launch_small(Block* b, int bn, const TcArgs& t, dim3 grid, size_t aux) {
  switch (bn) {
    case 16: launch_tc(b, Op<16>{t}, grid, aux); break;
    case 32: launch_tc(b, Op<32>{t}, grid, aux); break;
    case 48: launch_tc(b, Op<48>{t}, grid, aux); break;
    default: launch_tc(b, Op<64>{t}, grid, aux); break;
  }
}

static TcArgs make_args(const LayerArgs<float>& a) {
  TcArgs t{};
  t.a = a;
  t.kp = round_up(a.k, 8);
  t.vec = (a.C % 4 == 0) && (a.Ca % 4 == 0) && (a.c % 4 == 0);
  return t;
}

static unsigned mtiles(int64_t rows) { return static_cast<unsigned>((rows + tc::kBM - 1) / tc::kBM); }

void tc_conv1x1_fwd(Block* b, const LayerArgs<float>& a) {
  const TcArgs t = make_args(a);
  launch_bn<tc::Tc1x1Fwd>(b, pick_bn(a.bk), t, dim3(mtiles(a.M)), sizeof(BnAff) * a.c);
}

// ---- 3x3 halo kernels ----------------------------------------------------------
template <class Op>
static void launch_halo(Block* b, const Op& op, dim3 grid, size_t stage, int nst, size_t aux) {
  launch(tc::tc_halo_kernel<Op>, grid, tc::kThreads, stage * nst + aux, b->stream, op);
}

static tc::HaloArgs halo_args(const LayerArgs<float>& a, int kc) {
  tc::HaloArgs h{};
  h.a = a;
  h.g = tc::HaloGeom::make(a.H, a.W);
  h.kc = kc;
  h.vec = (a.C % 4 == 0) && (a.Ca % 4 == 0) && (a.c % 4 == 0);
  return h;
}

static int64_t nimg(const LayerArgs<float>& a) { return a.M / (static_cast<int64_t>(a.H) * a.W); }
static constexpr size_t kHaloSmemMax = 220 * 1024;

// Static choice of the halo kernels' tiles for a block (shared by the arena
// plan, the weight pre-tiling and the launches).
HaloPlan tc_halo_plan(const dpb_block_desc& d) {
  HaloPlan p{};
  const tc::HaloGeom g = tc::HaloGeom::make(static_cast<int>(d.h), static_cast<int>(d.w));
  const int bn = pick_bn(d.k);
  // The largest K chunk whose double-buffered stages let two CTAs share an SM
  // (the per-CTA produce -> MMA -> epilogue chain is latency-bound: a second
  // resident CTA overlaps it) for multi-wave grids, else the largest that
  // fits one CTA.
  // DPB_HALO_KC=<kc> forces a chunk (when it fits).
  static const int force_kc = std::getenv("DPB_HALO_KC") ? std::atoi(std::getenv("DPB_HALO_KC")) : 0;
  int ring = 2;  // raw halo ring depth of the forward producer
  auto fwd_aux = [&](int kc) {  // BN table + the raw fp32 halo ring (Tc3x3FwdHalo::fetch)
    using Op = tc::Tc3x3FwdHalo<16>;
    return static_cast<size_t>(Op::aux_bytes(static_cast<int>(d.bk), g.R, kc, ring));
  };
  auto fwd_fits = [&](int kc, size_t lim) {
    const size_t stage = 2ull * (static_cast<size_t>(g.R) * kc * 2 + 9ull * bn * kc * 2);
    const int nkb = (d.bk + kc - 1) / kc;
    return stage * (nkb > 1 ? 2 : 1) + fwd_aux(kc) <= lim;
  };
  int kc_pick = 0;
  // only when the tiles fill more than one wave at one CTA per SM (measured:
  // 56x56 and 28x28 gain 16 % / 10 %; 14x14 and 7x7, under one wave, lose to
  // the smaller chunks' extra rounds)
  const int64_t tiles = d.n * g.tpi;
  // (two CTAs per SM first with the two-slot raw ring, then with one slot)
  for (int want = 2; want >= 1 && !kc_pick; --want) {
    ring = want;
    for (int kc = std::min(64, d.bk); d.bk % 16 == 0 && bn <= 64 && kc >= 16 && !kc_pick && tiles > 148; kc /= 2)
      if (kc % 16 == 0 && fwd_fits(kc, kHaloSmemMax / 2 - 1024)) kc_pick = kc;
  }
  if (!kc_pick) ring = 2;
  if (force_kc >= 16 && force_kc % 16 == 0 && force_kc <= 64 && fwd_fits(force_kc, kHaloSmemMax)) kc_pick = force_kc;
  for (int kc = std::min(64, d.bk); d.bk % 16 == 0 && bn <= 64 && kc >= 16; kc /= 2) {
    if (kc % 16 != 0) continue;
    if (kc_pick && kc != kc_pick) continue;
    const size_t stage = 2ull * (static_cast<size_t>(g.R) * kc * 2 + 9ull * bn * kc * 2);
    const int nkb = (d.bk + kc - 1) / kc;
    const int nst = nkb > 1 ? 2 : 1;
    if (stage * nst + fwd_aux(kc) <= kHaloSmemMax) {
      p.fwd_ok = true;
      p.fwd_bn = bn;
      p.fwd_kc = kc;
      p.fwd_ring = ring;
      // under half a wave of tiles, a CTA pair per tile (cluster (1, 2), DSMEM
      // sum of the two K halves) when its exchange buffer fits too
      static const bool no_pair = std::getenv("DPB_HALO_NO_KPAIR") != nullptr;
      const bool taps = bn == 16 && d.k % 4 == 0 && 9 * d.k <= 128 && g.R <= 2 * tc::kBM;
      p.fwd_kpair = !no_pair && !taps && 2 * tiles <= 148 && nkb >= 2 && nkb % 2 == 0 &&
                    stage * nst + fwd_aux(kc) + 16 + static_cast<size_t>(tc::kBM) * bn * 4 <= kHaloSmemMax;
      p.fwd_layer_bytes = static_cast<int64_t>(nkb) * 2 * (9LL * bn * kc * 2);
      // all taps as GEMM columns: N = 9k <= 128 (two 128-column accumulators),
      // 4-column TMEM loads per tap, both 128-row M blocks inside the halo
      p.fwd_taps = bn == 16 && d.k % 4 == 0 && 9 * d.k <= 128 && g.R <= 2 * tc::kBM;
      break;
    }
  }
  int bnd = pick_bn(d.bk);
  const int kcd = round_up(d.k, 16);
  // under two waves of tiles, 64-column groups per tile (grid.y): twice the
  // CTAs, each with half the epilogue (the dgrad's epilogue is its longest
  // phase and is latency-bound at one CTA per SM)
  if (d.bk > 64 && d.bk % 64 == 0 && d.n * g.tpi <= 2 * 148) {
    p.bwd_split = static_cast<int>(d.bk / 64);
    bnd = 64;
  }
  const size_t stage_d = static_cast<size_t>(g.R) * kcd * 2 + 9ull * bnd * kcd * 2;
  if (kcd <= 64 && stage_d + sizeof(BnFwd) * d.bk <= kHaloSmemMax) {
    p.bwd_ok = true;
    p.bwd_bn = bnd;
    p.bwd_kc = kcd;
    p.bwd_layer_bytes = 9LL * bnd * kcd * 2 * p.bwd_split;
  }
  return p;
}

void tc_pretile_w2(Block* b, const float* params, bool fwd) {
  const dpb_block_desc& d = b->d;
  const HaloPlan& p = b->halo;
  const dim3 grid(8, d.m);
  if (fwd && p.fwd_ok && b->w2f && p.fwd_taps) {
    const int np = (9 * d.k + 15) / 16 * 16;
    launch(tc::k_pretile_w2_taps, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.fwd_kc, np,
                                                        p.fwd_layer_bytes, b->w2f);
    b->launches++;
  } else if (fwd && p.fwd_ok && b->w2f) {
    switch (p.fwd_bn) {
      case 16: launch(tc::k_pretile_w2_fwd<16>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.fwd_kc, b->w2f); break;
      case 32: launch(tc::k_pretile_w2_fwd<32>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.fwd_kc, b->w2f); break;
      case 48: launch(tc::k_pretile_w2_fwd<48>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.fwd_kc, b->w2f); break;
      default: launch(tc::k_pretile_w2_fwd<64>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.fwd_kc, b->w2f); break;
    }
    b->launches++;
  }
  if (!fwd && p.bwd_ok && b->w2b) {
    switch (p.bwd_bn) {
      case 16: launch(tc::k_pretile_w2_bwd<16>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.bwd_kc, p.bwd_split, b->w2b); break;
      case 32: launch(tc::k_pretile_w2_bwd<32>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.bwd_kc, p.bwd_split, b->w2b); break;
      case 48: launch(tc::k_pretile_w2_bwd<48>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.bwd_kc, p.bwd_split, b->w2b); break;
      case 64: launch(tc::k_pretile_w2_bwd<64>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.bwd_kc, p.bwd_split, b->w2b); break;
      case 128: launch(tc::k_pretile_w2_bwd<128>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.bwd_kc, p.bwd_split, b->w2b); break;
      case 192: launch(tc::k_pretile_w2_bwd<192>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.bwd_kc, p.bwd_split, b->w2b); break;
      default: launch(tc::k_pretile_w2_bwd<256>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, p.bwd_kc, p.bwd_split, b->w2b); break;
    }
    b->launches++;
  }
}

template <int BN>
static tc::Tc3x3FwdHalo<BN> fwd_op(const tc::HaloArgs& h, int ring) {
  tc::Tc3x3FwdHalo<BN> op{h};
  op.raw_want = ring;
  return op;
}

// Returns the number of per-CTA partial rows written (for the finalize).
int tc_conv3x3_fwd(Block* b, const LayerArgs<float>& a, int l) {
  const int bn = pick_bn(a.k);
  if (b->halo.fwd_ok && b->w2f) {
    const int kc = b->halo.fwd_kc;
    tc::HaloArgs h = halo_args(a, kc);
    h.wt = b->w2f + static_cast<int64_t>(l) * b->halo.fwd_layer_bytes;
    const size_t stage = 2ull * (static_cast<size_t>(h.g.R) * kc * 2 + 9ull * bn * kc * 2);
    const int nst = (a.bk + kc - 1) / kc > 1 ? 2 : 1;
    using FH = tc::Tc3x3FwdHalo<16>;
    const int ring = b->halo.fwd_ring;
    const size_t aux = FH::aux_bytes(a.bk, h.g.R, kc, ring);
    if (b->halo.fwd_taps) {
      const dim3 grid(static_cast<unsigned>(nimg(a) * h.g.tpi));
      const size_t np = (9 * a.k + 15) / 16 * 16;
      const size_t tstage = 2ull * (static_cast<size_t>(h.g.R) * kc * 2 + np * kc * 2);
      // the epilogue's per-tap output slices [9][128][k] fp32 reuse the stages
      const size_t ytap = 9ull * tc::kBM * a.k * 4;
      const size_t taux = std::max(aux, ytap > tstage * nst ? ytap - tstage * nst : size_t{0});
      tc::Tc3x3FwdTaps op{h};
      op.prod0 = 0;  // every warp produces (the taps GEMM keeps the shared-barrier engine path)
      op.raw_want = ring;
      launch_halo(b, op, grid, tstage, nst, taux);
      return static_cast<int>(grid.x);
    }
    if (b->halo.fwd_kpair) {
      const dim3 grid(static_cast<unsigned>(nimg(a) * h.g.tpi), 2);
      const size_t paux = (aux + 15) / 16 * 16 + static_cast<size_t>(tc::kBM) * bn * 4;
      auto go = [&](auto op) {
        op.kpair = 1;
        launch_cluster(tc::tc_halo_kernel<decltype(op)>, grid, tc::kThreads, stage * nst + paux, b->stream,
                       dim3(1, 2, 1), op);
      };
      switch (bn) {
        case 16: go(fwd_op<16>(h, ring)); break;
        case 32: go(fwd_op<32>(h, ring)); break;
        case 48: go(fwd_op<48>(h, ring)); break;
        default: go(fwd_op<64>(h, ring)); break;
      }
      return static_cast<int>(grid.x);
    }
    {
      const dim3 grid(static_cast<unsigned>(nimg(a) * h.g.tpi));
      switch (bn) {
        case 16: launch_halo(b, fwd_op<16>(h, ring), grid, stage, nst, aux); break;
        case 32: launch_halo(b, fwd_op<32>(h, ring), grid, stage, nst, aux); break;
        case 48: launch_halo(b, fwd_op<48>(h, ring), grid, stage, nst, aux); break;
        default: launch_halo(b, fwd_op<64>(h, ring), grid, stage, nst, aux); break;
      }
      return static_cast<int>(grid.x);
    }
  }
  const TcArgs t = make_args(a);
  launch_small<tc::Tc3x3Fwd>(b, bn, t, dim3(mtiles(a.M)),
                             sizeof(BnFwd) * a.bk + sizeof(int) * tc::kBM);
  return static_cast<int>(mtiles(a.M));
}

int tc_conv3x3_dgrad(Block* b, const LayerArgs<float>& a, int l) {
  const int bn = b->halo.bwd_ok ? b->halo.bwd_bn : pick_bn(a.bk);
  const int kc = round_up(a.k, 16);
  if (b->halo.bwd_ok && b->w2b) {
    tc::HaloArgs h = halo_args(a, kc);
    h.wt = b->w2b + static_cast<int64_t>(l) * b->halo.bwd_layer_bytes;
    const size_t stage = static_cast<size_t>(h.g.R) * kc * 2 + 9ull * bn * kc * 2;
    const size_t aux = sizeof(BnFwd) * a.bk;
    {
      const dim3 grid(static_cast<unsigned>(nimg(a) * h.g.tpi), static_cast<unsigned>(b->halo.bwd_split));
      switch (bn) {
        case 16: launch_halo(b, tc::Tc3x3DgradHalo<16>{h}, grid, stage, 1, aux); break;
        case 32: launch_halo(b, tc::Tc3x3DgradHalo<32>{h}, grid, stage, 1, aux); break;
        case 48: launch_halo(b, tc::Tc3x3DgradHalo<48>{h}, grid, stage, 1, aux); break;
        case 64: launch_halo(b, tc::Tc3x3DgradHalo<64>{h}, grid, stage, 1, aux); break;
        case 128: launch_halo(b, tc::Tc3x3DgradHalo<128>{h}, grid, stage, 1, aux); break;
        case 192: launch_halo(b, tc::Tc3x3DgradHalo<192>{h}, grid, stage, 1, aux); break;
        default: launch_halo(b, tc::Tc3x3DgradHalo<256>{h}, grid, stage, 1, aux); break;
      }
      return static_cast<int>(grid.x);
    }
  }
  const TcArgs t = make_args(a);
  launch_bn<tc::Tc3x3Dgrad>(b, bn, t, dim3(mtiles(a.M)),
                            sizeof(BnFwd) * a.bk + sizeof(int) * tc::kBM);
  return static_cast<int>(mtiles(a.M));
}

int64_t tc_halo_partials(const dpb_block_desc& d) {
  const tc::HaloGeom g = tc::HaloGeom::make(static_cast<int>(d.h), static_cast<int>(d.w));
  return d.n * g.tpi;
}

// split count of the halo 3x3 wgrad for a block (used by the arena plan)
// CTAs (tile ranges x channel groups) of the 3x3 wgrad; DPB_WGRAD3_CTAS overrides
static int64_t wgrad3_target() {
  static const int64_t t = std::getenv("DPB_WGRAD3_CTAS") ? std::atoll(std::getenv("DPB_WGRAD3_CTAS")) : 296;
  return t;
}
int64_t tc_halo_wgrad_splits(const dpb_block_desc& d) {
  const tc::HaloGeom g = tc::HaloGeom::make(static_cast<int>(d.h), static_cast<int>(d.w));
  const int64_t ntiles = d.n * g.tpi;
  const int64_t gy = (d.bk + tc::kBM - 1) / tc::kBM;
  const int64_t target = std::max<int64_t>(1, wgrad3_target() / gy);
  const int64_t tpc = std::max<int64_t>(1, (ntiles + target - 1) / target);
  return (ntiles + tpc - 1) / tpc;
}

void tc_conv1x1_dgrad(Block* b, const LayerArgs<float>& a) {
  const TcArgs t = make_args(a);
  const int bn = a.c <= 64 ? 64 : 128;
  const size_t aux = (sizeof(BnBwd) * a.bk + 15) / 16 * 16 + sizeof(BnFwd) * bn;
  const dim3 grid(mtiles(a.M), static_cast<unsigned>((a.c + bn - 1) / bn));
  if (bn == 64) launch_tc(b, tc::Tc1x1Dgrad<64>{t}, grid, aux);
  else launch_tc(b, tc::Tc1x1Dgrad<128>{t}, grid, aux);
}

// Split-K over pixels for the weight gradients: ~2 waves of 148 SMs, chunks
// a multiple of the K block and at least one K block (small M: many short
// splits rather than a few long latency chains).
int64_t tc_wgrad_chunk(int64_t M, int64_t tiles) {
  int64_t splits = std::max<int64_t>(1, 296 / std::max<int64_t>(1, tiles));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, M / tc::kBK));
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
  {
    const int bn = pick_bn(a.k);
    const tc::HaloArgs h = halo_args(a, bn);
    const size_t stage = static_cast<size_t>(h.g.R) * tc::kBM * 2 + static_cast<size_t>(tc::kBM) * bn * 2;
    const size_t aux = tc::Tc3x3WgradHalo<16>::aux_bytes(a.bk, h.g.R);
    if (bn <= 48 && 2 * stage + aux <= kHaloSmemMax) {
      const int64_t ntiles = nimg(a) * h.g.tpi;
      const int64_t gy = (a.bk + tc::kBM - 1) / tc::kBM;
      const int64_t target = std::max<int64_t>(1, wgrad3_target() / gy);
      const int tpc = static_cast<int>(std::max<int64_t>(1, (ntiles + target - 1) / target));
      const int gx = static_cast<int>((ntiles + tpc - 1) / tpc);
      const dim3 grid(gx, static_cast<unsigned>(gy));
      const int nst = tpc > 1 ? 2 : 1;
      switch (bn) {
        case 16: launch_halo(b, tc::Tc3x3WgradHalo<16>{h, tpc, static_cast<int>(ntiles)}, grid, stage, nst, aux); break;
        case 32: launch_halo(b, tc::Tc3x3WgradHalo<32>{h, tpc, static_cast<int>(ntiles)}, grid, stage, nst, aux); break;
        default: launch_halo(b, tc::Tc3x3WgradHalo<48>{h, tpc, static_cast<int>(ntiles)}, grid, stage, nst, aux); break;
      }
      return gx;
    }
  }
  const int64_t tiles = mtiles(9LL * a.bk);
  a.kchunk = tc_wgrad_chunk(a.M, tiles);
  const int splits = static_cast<int>((a.M + a.kchunk - 1) / a.kchunk);
  const TcArgs t = make_args(a);
  launch_small<tc::Tc3x3Wgrad>(b, pick_bn(a.k), t, dim3(mtiles(9LL * a.bk), 1, splits),
                               sizeof(BnFwd) * a.bk);
  return splits;
}

}  // namespace dpb

// Debug-only (not part of dpb.h): enable / read the halo engine's phase clocks.
extern "C" __attribute__((visibility("default"))) int dpb_debug_phase_clocks(int enable, long long* host,
                                                                             int n) {
  if (enable >= 0) {
    const int on = enable & 0xFFFF;
    cudaMemcpyToSymbol(dpb::tc::g_phase_on, &on, sizeof(int));
    return 0;
  }
  if (n < 0)  // per-K-chunk stamps: [cta][8][4]
    return cudaMemcpyFromSymbol(host, dpb::tc::g_kb_clock, sizeof(long long) * 32 * (-n));
  return cudaMemcpyFromSymbol(host, dpb::tc::g_phase_clock, sizeof(long long) * 9 * n);
}
