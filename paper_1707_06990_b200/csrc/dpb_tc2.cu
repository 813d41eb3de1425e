// Launchers of the persistent TMA-fed engine (dpb_tc2.cuh) and the host-side
// TMA tensor-map encoding (driver entry point cuTensorMapEncodeTiled).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "dpb_internal.h"
#include "dpb_launch.h"
#include "dpb_tc2.cuh"

namespace dpb {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D fp32 tensor map over rows x cols (row pitch in elements), box
// {box_cols, box_rows}, 128-byte swizzle, zero fill out of bounds.
bool make_map_f32(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t pitch,
                  int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || (pitch * 4) % 16 != 0) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * 4};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kPlanSms = 148;  // B200: the arena plan sizes the split-K partials for it

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <class Op>
static constexpr size_t fixed_smem() {
  return 1024 + Op::kNR * Op::kRawBytes + Op::kNS * Op::kOpBytes + Op::kNE * Op::kEpiBytes;
}

template <class Op>
static void launch2(Block* b, const Op& op, dim3 grid, size_t aux) {
  launch(tc2::tc2_kernel<Op>, grid, tc2::Roles<Op>::kThreads, fixed_smem<Op>() + aux, b->stream, op);
}

int tc2_bn_1x1(int bk) {
  const int n = (bk + 15) / 16 * 16;
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 48) return 48;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  if (n <= 192) return 192;
  return 0;
}

// bytes of the pre-tiled W1 operands of layer l (0 when unsupported)
int64_t tc2_w1_tile_bytes(const dpb_block_desc& d, int l) {
  const int bn = tc2_bn_1x1(d.bk);
  if (!bn) return 0;
  const int c = d.c0 + l * d.k;
  return static_cast<int64_t>((c + tc::kBK - 1) / tc::kBK) * 2 * (bn * tc::kBK * 2);
}

void tc2_pretile_w1(Block* b, const float* params) {
  const dpb_block_desc& d = b->d;
  const int bn = tc2_bn_1x1(d.bk);
  if (!bn || !b->wtile) return;
  const dim3 grid(16, d.m);
  switch (bn) {
    case 16: launch(tc2::k_pretile_w1_all<16>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 32: launch(tc2::k_pretile_w1_all<32>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 48: launch(tc2::k_pretile_w1_all<48>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 64: launch(tc2::k_pretile_w1_all<64>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 128: launch(tc2::k_pretile_w1_all<128>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    default: launch(tc2::k_pretile_w1_all<192>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, d.m, b->wtile); break;
  }
  b->launches++;
}

// Persistent CTAs for `ntiles` tiles on `slots` SMs: as many rounds as the
// full grid needs, but no more CTAs than those rounds require (512 tiles on
// 148 SMs: 128 CTAs x 4 tiles, not 148 CTAs of 3-4), so the SMs a short last
// round leaves idle are free for the other stream and the next launch.
// DPB_NO_BALANCE=1: one CTA per SM.
static int balanced_ctas(int ntiles, int slots) {
  static const bool off = std::getenv("DPB_NO_BALANCE") != nullptr;
  slots = std::max(1, slots);
  if (off) return std::max(1, std::min(ntiles, slots));
  const int rounds = (ntiles + slots - 1) / slots;
  return std::max(1, (ntiles + rounds - 1) / rounds);
}

// Column tiles per pixel tile for the streamed 1x1 forward over a W1 image of
// bimg columns: tiles of nw = bimg / ns columns (a multiple of 16, the MMA's N
// step, >= 32 and <= bnmax, the kernel's tile bound).  When the pixel tiles
// alone fill half the GPU, the fewest column tiles; otherwise the most that
// still fit one wave (ntiles * ns <= SMs).  0: no valid split.
// DPB_FWD_NO_SPLIT=1: the fewest column tiles always.
static int fwd1x1_col_split(int bimg, int bnmax, int ntiles, int sms) {
  static const bool off = std::getenv("DPB_FWD_NO_SPLIT") != nullptr;
  int lo = 0, best = 0;
  for (int ns = 1; ns <= 6; ++ns) {
    const int nw = bimg / ns;
    if (bimg % ns || nw % 16 || nw > bnmax || (ns > 1 && nw < 32)) continue;
    if (!lo) lo = ns;
    if (ntiles * ns <= sms) best = ns;
  }
  if (!lo) return 0;
  static const int force = std::getenv("DPB_FWD_NS") ? std::atoi(std::getenv("DPB_FWD_NS")) : 0;
  if (force >= lo && force <= 6 && bimg % force == 0 && (bimg / force) % 16 == 0 && bimg / force >= 32)
    return force;
  if (off || 2 * ntiles > sms || best < lo) return lo;
  return best;
}

// K splits of the streamed 1x1 forward for a layer with c input channels over
// M pixels: the split count minimising the persistent grid's makespan
// ceil(tiles * ks / SMs) / ks, taken when it beats no split by >= 25% and the
// tiles fill at most a quarter of the SMs (the partials' second pass costs a
// launch).  1 = no split.  DPB_FWD_NO_KSPLIT=1.
int tc2_fwd_ksplit(int64_t M, int c, int sms, int ns) {
  static const bool off = std::getenv("DPB_FWD_NO_KSPLIT") != nullptr;
  if (off) return 1;
  const int64_t nt = (M + tc::kBM - 1) / tc::kBM * ns;  // tiles before the split
  // measured: a win where the column split left the SMs starved (7x7 at batch
  // 64: 25 pixel tiles, 58 -> ~35 us per layer with the reduce), a loss at
  // 14x14 (98 tiles): the reduce pass costs more than the balance gains
  if (nt * 4 > sms) return 1;
  const int nkb = (c + tc::kBK - 1) / tc::kBK;
  int best = 1;
  double best_t = static_cast<double>((nt + sms - 1) / sms);
  for (int ks = 2; ks <= tc2::kMaxKSplit && ks <= nkb; ++ks) {
    const double t = static_cast<double>((nt * ks + sms - 1) / sms) / ks;
    if (t < best_t - 1e-9) {
      best_t = t;
      best = ks;
    }
  }
  const double t1 = static_cast<double>((nt + sms - 1) / sms);
  return best_t <= 0.75 * t1 ? best : 1;
}

static bool fwd_in_place() {  // DPB_FWD_NO_INPLACE=1: the two-stage ring with an operand ring
  static const bool on = std::getenv("DPB_FWD_NO_INPLACE") == nullptr;
  return on;
}

// 1x1 forward on the v2 engine; false when the shape is not supported (the
// caller then uses the v1 kernel).
bool tc2_conv1x1_fwd(Block* b, const LayerArgs<float>& a, int l, int* prows) {
  if (a.C % 4 != 0 || !b->wtile) return false;
  const int ntiles = static_cast<int>((a.M + tc::kBM - 1) / tc::kBM);
  const uint8_t* w1t = b->wtile + b->wtile_off[l];
  auto go = [&](auto tag) -> bool {
    using Op = decltype(tag);
    const int nkb = (a.c + tc::kBK - 1) / tc::kBK;
    const size_t aux = sizeof(BnAff) * a.c + (Op::kMmaReadsRaw ? 0 : nkb * 2 * Op::kBBytes);
    if (fixed_smem<Op>() + aux > 220 * 1024) return false;
    Op op{};
    if (!make_map_f32(&op.xmap, a.feat, a.C, a.M, a.C, 32, tc::kBM)) return false;
    op.a = a;
    op.w1t = w1t;
    if constexpr (Op::kMmaReadsRaw) {  // streamed W1: split-K or column-split small blocks
      op.bimg = tc2_bn_1x1(a.bk);
      // split-K over the narrowest column split the stage width allows
      const int ns0 = (op.bimg + Op::BN - 1) / Op::BN;
      const bool ok0 = op.bimg % ns0 == 0 && (op.bimg / ns0) % 16 == 0;
      const int ks = (b->zpart && ok0) ? tc2_fwd_ksplit(a.M, a.c, kPlanSms, ns0) : 1;
      if (ks > 1) {
        op.kper = (nkb + ks - 1) / ks;
        op.ks = (nkb + op.kper - 1) / op.kper;  // every split holds >= 1 K block
        op.zpart = b->zpart;
        op.ns = ns0;
      } else {
        op.ns = fwd1x1_col_split(op.bimg, Op::BN, ntiles, num_sms());
        if (!op.ns) return false;
      }
      op.nw = op.bimg / op.ns;
    }
    launch2(b, op, dim3(balanced_ctas(ntiles * op.ns * op.ks, num_sms())), aux);
    if (op.ks > 1) {
      const int zb = static_cast<int>((a.M + tc2::kZRows - 1) / tc2::kZRows);
      launch(tc2::k_zsplit_reduce, dim3(zb, (a.bk + 31) / 32), 256, 0, b->stream,
             static_cast<const float*>(b->zpart), op.ks, a.M, a.bk, a.z, a.part);
      if (prows) *prows = zb;
    }
    return true;
  };
  // B resident in shared memory when all of W1's tiles fit, else streamed
  switch (tc2_bn_1x1(a.bk)) {
    case 16: return go(tc2::Fwd1x1<16, true>{}) || go(tc2::Fwd1x1<16, false>{});
    case 32: return go(tc2::Fwd1x1<32, true>{}) || go(tc2::Fwd1x1<32, false>{});
    case 48: return go(tc2::Fwd1x1<48, true>{}) || go(tc2::Fwd1x1<48, false>{});
    case 64: return go(tc2::Fwd1x1<64, true>{}) || go(tc2::Fwd1x1<64, false>{});
    // wide inputs: W1's streamed stage at the full width no longer fits beside
    // the BN table, so the stages hold half-width (or narrower) column tiles
    case 128: return go(tc2::Fwd1x1<128, true>{}) || (fwd_in_place() && go(tc2::Fwd1x1<128, false, true>{})) ||
                     go(tc2::Fwd1x1<128, false>{}) || go(tc2::Fwd1x1<64, false>{});
    case 192: return go(tc2::Fwd1x1<192, true>{}) || go(tc2::Fwd1x1<192, false>{}) ||
                     go(tc2::Fwd1x1<96, false>{});
    default: return false;
  }
}

// ---- 1x1 backward data on the v2 engine ------------------------------------------
// Column-tile width bound of Dgrad1x1 for a block (0: not supported).
// 128 columns: its two TMEM accumulators then take 256 of the SM's 512 columns,
// so a CTA can start beside a side-stream 3x3 wgrad CTA (which holds 256)
// instead of waiting for the SM to empty (measured +0.6 % over 256 at BC-100).
// (256-column tiles for wide blocks, forming t1 half as often, were tried:
// the 64 KB W1^T image leaves room for only a 3-deep epilogue ring, fewer
// boxes than the four epilogue groups need in flight — it stalls.)
int tc2_bwd_bn(const dpb_block_desc&) { return 128; }

int64_t tc2_w1b_layer_bytes(const dpb_block_desc& d, int l) {
  const int bn = tc2_bwd_bn(d);
  int nn, nw;
  tc2::bwd_ntiles(d.c0 + l * d.k, bn, nn, nw);
  return static_cast<int64_t>(nn) * tc2::bwd_nkb(d.bk) * bn * 64;
}

void tc2_pretile_w1t(Block* b, const float* params) {
  const dpb_block_desc& d = b->d;
  if (!b->w1b) return;
  const dim3 grid(16, d.m);
  launch(tc2::k_pretile_w1t_all<128>, grid, 256, 0, b->stream, params, d.c0, d.k, d.bk, b->w1b);
  b->launches++;
}

bool tc2_conv1x1_dgrad(Block* b, const LayerArgs<float>& a, int l) {
  if (a.C % 4 != 0 || a.cg % 4 != 0 || !b->w1b) return false;
  const int ntiles = static_cast<int>((a.M + tc::kBM - 1) / tc::kBM);
  auto go = [&](auto tag) -> bool {
    using Op = decltype(tag);
    const size_t aux = static_cast<size_t>(tc2::bwd_nkb(a.bk)) * Op::kBTile +
                       (sizeof(BnBwd) * a.bk + 15) / 16 * 16 + sizeof(BnFwd) * Op::BN;
    if (fixed_smem<Op>() + aux > 222 * 1024) return false;  // + ~4 KB static: under the 227 KB opt-in
    Op op{};
    if (!make_map_f32(&op.gmap, a.g0, a.bk, a.M, a.bk, 32, tc::kBM) ||
        !make_map_f32(&op.zmap, a.z, a.bk, a.M, a.bk, 32, tc::kBM) ||
        !make_map_f32(&op.fmap, a.feat, a.C, a.M, a.C, 32, tc::kBM) ||
        !make_map_f32(&op.omap, a.g1, a.c, a.M, a.cg, 32, tc::kBM))
      return false;
    op.a = a;
    op.w1t = b->w1b + b->w1b_off[l];
    int nn, nw;
    tc2::bwd_ntiles(a.c, Op::BN, nn, nw);
    op.nw = nw;
    const int gx = balanced_ctas(ntiles, std::max(1, num_sms() / nn));
    launch2(b, op, dim3(gx, nn), aux);
    return true;
  };
  // bk = 192: the resident W1^T (48 KB) fits only beside a 4-deep epilogue ring
  static const int ne = std::getenv("DPB_DGRAD_NE") ? std::atoi(std::getenv("DPB_DGRAD_NE")) : 7;
  return (ne >= 7 && go(tc2::Dgrad1x1<128, 7>{})) || (ne >= 6 && go(tc2::Dgrad1x1<128, 6>{})) ||
         go(tc2::Dgrad1x1<128>{}) || go(tc2::Dgrad1x1<128, 4>{});
}

// ---- 1x1 backward weights on the v2 engine -----------------------------------------
// Upper bound of the split count (CTAs along x) for the arena plan.
int64_t tc2_wgrad_wpart_elems(const dpb_block_desc& d, int l) {
  const int c = d.c0 + l * d.k;
  const int bn = d.bk <= 64 ? 256 : 128;
  int nn, nw;
  tc2::bwd_ntiles(c, bn, nn, nw);
  return static_cast<int64_t>(std::max(1, 160 / nn)) * d.bk * c;
}

// Returns the number of splits written to wpart ([split][j][i]), 0 when the
// shape is not supported (the caller then uses the v1 kernel).
int tc2_conv1x1_wgrad(Block* b, const LayerArgs<float>& a) {
  if (a.C % 4 != 0 || a.bk % 8 != 0 || a.bk > 192) return 0;
  int splits = 0;
  auto go = [&](auto tag) -> bool {
    using Op = decltype(tag);
    const size_t aux = (sizeof(BnBwd) * a.bk + 15) / 16 * 16 + sizeof(BnFwd) * Op::BN;
    if (fixed_smem<Op>() + aux > 220 * 1024) return false;
    Op op{};
    if (!make_map_f32(&op.gmap, a.g0, a.bk, a.M, a.bk, 32, Op::kBoxP) ||
        !make_map_f32(&op.zmap, a.z, a.bk, a.M, a.bk, 32, Op::kBoxP) ||
        !make_map_f32(&op.fmap, a.feat, a.C, a.M, a.C, 32, Op::kBoxP))
      return false;
    op.a = a;
    int nn, nw;
    tc2::bwd_ntiles(a.c, Op::BN, nn, nw);
    op.nw = nw;
    op.nblk = static_cast<int>((a.M + Op::kBoxP - 1) / Op::kBoxP);
    // Half the SMs at bk <= 64: this runs on the side stream next to the
    // data-gradient chain, and a smaller footprint leaves that chain its SMs
    // (measured +1.5 % over one CTA per SM at BC-100; a quarter is slower
    // again).  At bk >= 128 (DenseNet-121/264) the weight branch carries more
    // work per pixel and every SM pays: +5 % at d121, +8 % at d264k48 over
    // half.  DPB_WGRAD_SM_DIV=<d>: 1/d of the SMs for every shape.
    static const char* env_div = std::getenv("DPB_WGRAD_SM_DIV");
    const int div = env_div ? std::max(1, std::atoi(env_div)) : (a.bk <= 64 ? 2 : 1);
    const int target = std::max(1, num_sms() / (div * nn));
    op.kchunk = (op.nblk + target - 1) / target;
    const int gx = (op.nblk + op.kchunk - 1) / op.kchunk;  // every CTA owns >= 1 block
    launch2(b, op, dim3(gx, nn), aux);
    splits = gx;
    return true;
  };
  const int jb = (a.bk + 31) / 32;
  const bool ok = jb <= 2 ? go(tc2::Wgrad1x1<256, 2>{})
                  : jb <= 4 ? go(tc2::Wgrad1x1<128, 4>{})
                            : go(tc2::Wgrad1x1<128, 6>{});
  return ok ? splits : 0;
}

}  // namespace dpb

// Debug-only (not part of dpb.h): arm the v2 engine's phase clocks for launches
// with layer width c (c <= 0 disarms), or read them (host: 148 x 28 int64).
extern "C" __attribute__((visibility("default"))) int dpb_debug_tc2_clocks(int c, long long* host) {
  if (host == nullptr) {
    c &= 0xffff;
    return cudaMemcpyToSymbol(dpb::tc2::g_tc2_dbg_c, &c, sizeof(int));
  }
  return cudaMemcpyFromSymbol(host, dpb::tc2::g_tc2_clock, sizeof(long long) * 148 * 28);
}
