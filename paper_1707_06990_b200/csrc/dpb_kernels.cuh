// Elementwise / reduction kernels of the dense block (HBM-bound work).
#pragma once

#include "dpb_common.cuh"

namespace dpb {

// --- layout conversion at the reference-facing boundary ----------------------
// NCHW fp32 [n, c, h, w] (sample stride c*h*w) <-> NHWC rows of pitch P at
// channel offset c_off.  32x32 shared-memory transpose tiles: coalesced on
// both sides.
template <typename S>
__global__ void k_nchw_to_nhwc(const float* __restrict__ src, int64_t n, int c,
                               int64_t hw, S* __restrict__ dst, int pitch,
                               int c_off) {
  pdl_enter();
  __shared__ float tile[32][33];
  const int64_t img = blockIdx.z;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int c0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int ch = c0 + r;
    const int64_t p = p0 + threadIdx.x;
    if (ch < c && p < hw) tile[r][threadIdx.x] = src[(img * c + ch) * hw + p];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t p = p0 + r;
    const int ch = c0 + threadIdx.x;
    if (ch < c && p < hw) dst[(img * hw + p) * pitch + c_off + ch] = from_f<S>(tile[threadIdx.x][r]);
  }
}

template <typename S>
__global__ void k_nhwc_to_nchw(const S* __restrict__ src, int pitch, int c_off,
                               int64_t n, int c, int64_t hw,
                               float* __restrict__ dst) {
  pdl_enter();
  __shared__ float tile[32][33];
  const int64_t img = blockIdx.z;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int c0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t p = p0 + r;
    const int ch = c0 + threadIdx.x;
    if (ch < c && p < hw) tile[threadIdx.x][r] = to_f(src[(img * hw + p) * pitch + c_off + ch]);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int ch = c0 + r;
    const int64_t p = p0 + threadIdx.x;
    if (ch < c && p < hw) dst[(img * c + ch) * hw + p] = tile[r][threadIdx.x];
  }
}

// NHWC strided copy (c channels of pitch sp at offset so) -> (pitch dp, off do)
template <typename S>
__global__ void k_nhwc_copy(const float* __restrict__ src, int sp, int64_t M, int c,
                            S* __restrict__ dst, int dp, int d_off) {
  pdl_enter();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= M * c) return;
  const int64_t p = i / c;
  const int ch = static_cast<int>(i - p * c);
  dst[p * dp + d_off + ch] = from_f<S>(src[p * sp + ch]);
}

// --- per-channel partial sums over rows of an NHWC buffer -------------------
// grid.x = ceil(M / 128) CTAs (the same partial count as the GEMM epilogues),
// grid.y = groups of 32 channels (wide block inputs at small M: block 4 of
// DenseNet-264 has 25 row CTAs and 1,152-1,728 channels); 256 threads = 8 row
// groups x 32 channel lanes.  Writes part[cta][ch] =
// {sum x, sum x^2} in fp64.
template <typename S>
__global__ void __launch_bounds__(256)
k_channel_partials(const S* __restrict__ src, int pitch, int c_off, int64_t M,
                   int nch, double2* __restrict__ part) {
  pdl_enter();
  __shared__ double r1[8][33], r2[8][33];
  const int lane = threadIdx.x % 32, grp = threadIdx.x / 32;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * 128;
  for (int cb = blockIdx.y * 32; cb < nch; cb += 32 * gridDim.y) {  // grid.y: channel groups
    const int ch = cb + lane;
    double s1 = 0.0, s2 = 0.0;
    if (ch < nch) {
      for (int r = grp; r < 128; r += 8) {
        const int64_t m = m0 + r;
        if (m >= M) break;
        const double v = to_f(src[m * pitch + c_off + ch]);
        s1 += v;
        s2 += v * v;
      }
    }
    r1[grp][lane] = s1;
    r2[grp][lane] = s2;
    __syncthreads();
    if (grp == 0 && ch < nch) {
      double a = 0.0, b = 0.0;
      for (int g = 0; g < 8; ++g) { a += r1[g][lane]; b += r2[g][lane]; }
      part[static_cast<int64_t>(blockIdx.x) * nch + ch] = make_double2(a, b);
    }
    __syncthreads();
  }
}

// Block-wide fixed-order fold for the finalize kernels: a CTA of kFinThreads
// owns kFinCh channels; thread (lane, ch) sums partials p = lane, lane +
// kFinLanes, ... (each row read is kFinCh consecutive double2: coalesced), then
// thread (0, ch) adds the kFinLanes sums in lane order.  Deterministic; at most
// ~P / 64 loads per thread, all independent (the finalize sits on the
// critical path between two big kernels, so its latency is what matters).
constexpr int kFinCh = 16, kFinLanes = 64, kFinThreads = kFinCh * kFinLanes;
// CH channels per CTA (kFinCh, or 4 when there are many partial rows: four
// times the CTAs pulling them), kFinThreads / CH lanes.  The lane sums are
// added in lane order (CH = kFinCh), or in 16 runs of 16 lanes then the 16
// run sums in order (CH = 4): fixed either way.
template <int CH>
__device__ __forceinline__ bool fold_block(const double2* part, int P, int nch, int& ch, double2& out) {
  constexpr int L = kFinThreads / CH;
  __shared__ double2 red[L][CH + 1];
  const int tx = threadIdx.x % CH, ty = threadIdx.x / CH;
  ch = blockIdx.x * CH + tx;
  double a = 0.0, b = 0.0;
  if (ch < nch) {
#pragma unroll 9
    for (int p = ty; p < P; p += L) {
      const double2 v = part[static_cast<int64_t>(p) * nch + ch];
      a += v.x;
      b += v.y;
    }
  }
  red[ty][tx] = make_double2(a, b);
  __syncthreads();
  if constexpr (L > 64) {
    constexpr int R = L / 16;  // lanes per run
    if (ty < 16) {
      double sa = 0.0, sb = 0.0;
      for (int i = 0; i < R; ++i) {
        sa += red[ty * R + i][tx].x;
        sb += red[ty * R + i][tx].y;
      }
      __syncwarp();
      red[ty * R][tx] = make_double2(sa, sb);  // run sum in its first lane's slot
    }
    __syncthreads();
    if (ty != 0 || ch >= nch) return false;
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < 16; ++i) {
      sa += red[i * R][tx].x;
      sb += red[i * R][tx].y;
    }
    out = make_double2(sa, sb);
    return true;
  } else {
    if (ty != 0 || ch >= nch) return false;
    double sa = 0.0, sb = 0.0;
#pragma unroll 16
    for (int i = 0; i < L; ++i) {
      sa += red[i][tx].x;
      sb += red[i][tx].y;
    }
    out = make_double2(sa, sb);
    return true;
  }
}

// Forward statistics: mean = S1/count, biased var = S2/count - mean^2
// (ops.hpp:138-162 semantics) -> mean_out[first+ch], var_out[first+ch].
// Grid ceil(nch / CH) x kFinThreads.
template <int CH = kFinCh>
__global__ void __launch_bounds__(kFinThreads) k_finalize_stats(const double2* __restrict__ part, int P, int nch,
                                 double count, float* __restrict__ mean_out,
                                 float* __restrict__ var_out, int first) {
  pdl_enter();
  int ch;
  double2 s;
  if (fold_block<CH>(part, P, nch, ch, s)) {
    const double mean = s.x / count;
    double var = s.y / count - mean * mean;
    if (var < 0.0) var = 0.0;
    mean_out[first + ch] = static_cast<float>(mean);
    var_out[first + ch] = static_cast<float>(var);
  }
}

// BN backward sums -> dgamma = sum g*xhat, dbeta = sum g (written, ops.hpp:229-230)
// and the apply coefficients coef[2*ch] = mg, [2*ch+1] = mgx.
template <int CH = kFinCh>
__global__ void __launch_bounds__(kFinThreads) k_finalize_bn_bwd(const double2* __restrict__ part, int P, int nch,
                                  double count, float* __restrict__ dgamma,
                                  float* __restrict__ dbeta, float* __restrict__ coef) {
  pdl_enter();
  int ch;
  double2 s;
  if (fold_block<CH>(part, P, nch, ch, s)) {
    const float sum_g = static_cast<float>(s.x);
    const float sum_gx = static_cast<float>(s.y);
    dgamma[ch] = sum_gx;
    dbeta[ch] = sum_g;
    coef[2 * ch] = static_cast<float>(s.x / count);
    coef[2 * ch + 1] = static_cast<float>(s.y / count);
  }
}

// acc[:, 0:c] += (gamma*inv) * (t2 - mg - xhat*mgx)   (BN_a backward apply fused
// with the concat-backward accumulate, graph.hpp:929-941).  HBM-bound: reads
// t2 (fp32) and x, read-modify-writes acc.  One thread per 4 channels.
template <typename S>
__global__ void __launch_bounds__(256)
k_bn_apply_accumulate(int64_t M, int c_lo, int c, int C, int Ca, int cg, const S* __restrict__ feat,
                      const float* __restrict__ g1, const float* __restrict__ amean,
                      const float* __restrict__ avar,
                      const float* __restrict__ gamma, const float* __restrict__ coef,
                      float* __restrict__ acc) {
  pdl_enter();
  const int nc = c - c_lo;  // channels [c_lo, c)
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= M * nc) return;
  const int64_t p = i / nc;
  const int ch = c_lo + static_cast<int>(i - p * nc);
  const float mean = amean[ch];
  const float inv = bn_inv(avar[ch]);
  const float xh = (to_f(feat[p * C + ch]) - mean) * inv;
  const float g = g1[p * cg + ch];
  acc[p * Ca + ch] += gamma[ch] * inv * (g - coef[2 * ch] - xh * coef[2 * ch + 1]);
}

// As k_bn_apply_accumulate with 16-byte rows (feature pitch C, accumulator
// pitch Ca, g1 pitch cg all multiples of 4; fp32 storage): a thread owns one
// 4-channel quad for kRows consecutive pixels (coefficients computed once,
// 16-byte loads/stores, warps coalesced along the row).  The last quad of a
// layer with c % 4 != 0 updates only its channels < c.  kRows = 8 for wide
// launches; the narrow head on the main chain (k channels) takes 2 rows per
// thread so its few quads still fill the SMs (a 4x shorter latency chain).
constexpr int kApplyRows = 8, kApplyRowsNarrow = 2;
template <int kRows>
__global__ void __launch_bounds__(256)
k_bn_apply_accumulate4(int64_t M, int c_lo, int c, int C, int Ca, int cg, const float* __restrict__ feat,
                       const float* __restrict__ g1, const float* __restrict__ amean,
                       const float* __restrict__ avar, const float* __restrict__ gamma,
                       const float* __restrict__ coef, float* __restrict__ acc) {
  const int q0 = c_lo >> 2;  // channels [c_lo, c) (c_lo % 4 == 0)
  const int cq = ((c + 3) >> 2) - q0;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t pg = t / cq;
  const int q = q0 + static_cast<int>(t - pg * cq);
  const int64_t p0 = pg * kRows;
  if (p0 >= M) {
    pdl_enter();
    return;
  }
  const int ch = 4 * q;
  // Only the BN_a coefficients come from the predecessor (the finalize); g1 is
  // the 1x1 dgrad's output two launches back, and the features, statistics and
  // accumulator are older.  So the first rows are loaded before the
  // grid-dependency wait.
  const float4 mean = *reinterpret_cast<const float4*>(amean + ch);
  const float4 var = *reinterpret_cast<const float4*>(avar + ch);
  constexpr int kPre = kRows < 2 ? kRows : 2;
  float4 xp[kPre], gp[kPre];
#pragma unroll
  for (int i = 0; i < kPre; ++i) {
    const int64_t p = p0 + i < M ? p0 + i : p0;
    xp[i] = *reinterpret_cast<const float4*>(feat + p * C + ch);
    gp[i] = *reinterpret_cast<const float4*>(g1 + p * cg + ch);
  }
  pdl_enter();
  const float4 c01 = *reinterpret_cast<const float4*>(coef + 2 * ch);      // mg0 mgx0 mg1 mgx1
  const float4 c23 = *reinterpret_cast<const float4*>(coef + 2 * ch + 4);  // mg2 mgx2 mg3 mgx3
  const float m[4] = {mean.x, mean.y, mean.z, mean.w};
  const float inv[4] = {bn_inv(var.x), bn_inv(var.y), bn_inv(var.z), bn_inv(var.w)};
  const float mg[4] = {c01.x, c01.z, c23.x, c23.z};
  const float mgx[4] = {c01.y, c01.w, c23.y, c23.w};
  const int live = c - ch < 4 ? c - ch : 4;  // channels of this quad inside the layer
  float gi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) gi[e] = e < live ? gamma[ch + e] * inv[e] : 0.f;
  const int64_t pe = p0 + kRows < M ? p0 + kRows : M;
  auto row = [&](int64_t p, const float4 x4, const float4 g4) {
    const float x[4] = {x4.x, x4.y, x4.z, x4.w};
    const float g[4] = {g4.x, g4.y, g4.z, g4.w};
    float r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float xh = (x[e] - m[e]) * inv[e];
      r[e] = gi[e] * (g[e] - mg[e] - xh * mgx[e]);
    }
    float* arow = acc + p * Ca + ch;
    if (live == 4) {
      float4 a = *reinterpret_cast<float4*>(arow);
      a.x += r[0];
      a.y += r[1];
      a.z += r[2];
      a.w += r[3];
      *reinterpret_cast<float4*>(arow) = a;
    } else {  // last quad of a layer with c % 4 != 0: channels >= c belong to later layers
      for (int e = 0; e < live; ++e) arow[e] += r[e];
    }
  };
#pragma unroll
  for (int i = 0; i < kPre; ++i)
    if (p0 + i < pe) row(p0 + i, xp[i], gp[i]);
  for (int64_t p = p0 + kPre; p < pe; ++p)
    row(p, *reinterpret_cast<const float4*>(feat + p * C + ch), *reinterpret_cast<const float4*>(g1 + p * cg + ch));
}

// Split-K weight-gradient folds.  Block (32 x 8): 32 consecutive partial
// elements (coalesced) x 8 split groups; each thread sums its group's splits
// in order, then the 8 group sums are added in a fixed order — deterministic.
template <class Index>
__device__ __forceinline__ void fold_splits(const float* __restrict__ wpart, int splits,
                                            int64_t n, Index out_index, float* __restrict__ out) {
  __shared__ float red[8][33];
  const int64_t e = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  float s = 0.f;
  if (e < n) {
#pragma unroll 8
    for (int z = threadIdx.y; z < splits; z += 8) s += wpart[static_cast<int64_t>(z) * n + e];
  }
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && e < n) {
    float t = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += red[g][threadIdx.x];
    out[out_index(e)] = t;
  }
}

// dW2: partial element e = r*k + o with r = tap*bk + j -> flat W2[o][j][tap]
__global__ void k_reduce_w2(const float* __restrict__ wpart, int splits, int bk, int k,
                            float* __restrict__ dw2) {
  pdl_enter();
  const int64_t n = 9LL * bk * k;
  fold_splits(wpart, splits, n, [=] __device__(int64_t e) {
    const int o = static_cast<int>(e % k);
    const int r = static_cast<int>(e / k);
    const int tap = r / bk, j = r - tap * bk;
    return (static_cast<int64_t>(o) * bk + j) * 9 + tap;
  }, dw2);
}

// dW1 (SIMT partials [split][j][i]) -> flat W1[j][i]
__global__ void k_reduce_w1(const float* __restrict__ wpart, int splits, int bk, int c,
                            float* __restrict__ dw1) {
  pdl_enter();
  fold_splits(wpart, splits, static_cast<int64_t>(bk) * c, [] __device__(int64_t e) { return e; },
              dw1);
}

// dW1 from the tensor-core partials [split][i][j] -> flat W1[j][i]
__global__ void k_reduce_w1t(const float* __restrict__ wpart, int splits, int bk, int c,
                             float* __restrict__ dw1) {
  pdl_enter();
  fold_splits(wpart, splits, static_cast<int64_t>(bk) * c, [=] __device__(int64_t e) {
    const int64_t i = e / bk, j = e - i * bk;
    return j * c + i;
  }, dw1);
}

// Statistics layout in the arena: fstat = mean[C] | var[C] for the feature
// channels (shared by every BN_a that reads them, F6); zstat = per layer
// mean[bk] | var[bk].  `stat_at` maps an index of the flat reference layout
// (per layer mean_a[c] var_a[c] mean_b[bk] var_b[bk]) to its arena value.
__device__ __forceinline__ float stat_at(int m, int c0, int k, int bk, int C,
                                         const float* fstat, const float* zstat,
                                         int64_t i) {
  int64_t o = 0;
  for (int l = 0; l < m; ++l) {
    const int c = c0 + l * k;
    const int64_t sz = 2 * c + 2 * bk;
    if (i < o + sz) {
      const int64_t r = i - o;
      if (r < c) return fstat[r];
      if (r < 2 * c) return fstat[C + (r - c)];
      return zstat[static_cast<int64_t>(l) * 2 * bk + (r - 2 * c)];
    }
    o += sz;
  }
  return 0.f;
}

// Running-statistics update for every BN of the block (ops.hpp:185-194):
// rm = (1-m) rm + m mean ; rv = (1-m) rv + m var_biased.
__global__ void k_running_update(int m, int c0, int k, int bk, int C,
                                 const float* __restrict__ fstat,
                                 const float* __restrict__ zstat,
                                 float* __restrict__ running, int64_t total) {
  pdl_enter();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const float s = stat_at(m, c0, k, bk, C, fstat, zstat, i);
  running[i] = (1.0f - kMomentum) * running[i] + kMomentum * s;
}

// Flat statistics export in the reference layout.
__global__ void k_export_stats(int m, int c0, int k, int bk, int C,
                               const float* __restrict__ fstat,
                               const float* __restrict__ zstat, float* __restrict__ out,
                               int64_t total) {
  pdl_enter();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  out[i] = stat_at(m, c0, k, bk, C, fstat, zstat, i);
}

}  // namespace dpb
