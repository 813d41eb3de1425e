// Whole-network training step around the dense blocks:
// stem, transitions, head and loss of GraphPlan<T> (dp/graph.hpp:731-826,
// :1065-1183, ops dp/ops.hpp:392-560), on the GPU.  The dense blocks run
// through the block path (dpb_block.cu); everything here is small next to
// them (the transitions' 1x1 convs are ~3% of BC-100's FLOPs), so these
// kernels are plain fp32 CUDA-core code with fixed-order reductions
// (deterministic), except the transitions' forward and pooled-input-gradient
// GEMMs of the bf16 path (TransGemm on the tcgen05 engine, bf16x3 products).
// Activations are NHWC fp32 like the block arenas.
//
// Transition: BN (batch statistics of every feature channel are already in
// the block's arena, F6) -> ReLU -> 2x2 average pool -> 1x1 conv.  The
// reference convolves first and pools after (graph.hpp:774-782); both are
// linear per pixel, so pooling first is the same map on a quarter of the
// pixels.  Its backward mirrors that: dW from the pooled activations,
// the pooled-input gradient spread back over each 2x2 window.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "dpb_comm.h"
#include "dpb_common.cuh"
#include "dpb_internal.h"
#include "dpb_launch.h"
#include "dpb_tc.cuh"

struct dpb_model;

namespace dpb {
namespace {

constexpr float kMomentum = 0.1f;  // ops.hpp batchnorm_forward running update

__device__ __forceinline__ float bn_ref(float x, float mean, float inv, float gamma, float beta) {
  // the reference's expression gamma * (x - mean) * inv + beta (ops.hpp:130)
  return __fadd_rn(__fmul_rn(__fmul_rn(gamma, __fsub_rn(x, mean)), inv), beta);
}

// ---- stem: conv3x3, stride 1, pad 1 (graph.hpp:739-742) ----------------------------
// in NCHW [N, cin, H, W] -> out NHWC rows of pitch `ld` (channels [0, c0)).
__global__ void k_stem_fwd(const float* __restrict__ in, int64_t N, int cin, int H, int W,
                           const float* __restrict__ w, int c0, float* __restrict__ out, int ld) {
  pdl_enter();
  extern __shared__ float ws[];  // c0 x cin x 9 weights
  for (int i = threadIdx.x; i < c0 * cin * 9; i += blockDim.x) ws[i] = w[i];
  __syncthreads();
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= N * H * W) return;
  const int hw = H * W;
  const int n = static_cast<int>(p / hw);
  const int rem = static_cast<int>(p - static_cast<int64_t>(n) * hw);
  const int y = rem / W, x = rem - (rem / W) * W;
  float win[4 * 9];  // cin <= 4 (dpb_model_create)
  for (int ci = 0; ci < cin; ++ci)
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int yy = y + t / 3 - 1, xx = x + t % 3 - 1;
      win[ci * 9 + t] = (yy >= 0 && yy < H && xx >= 0 && xx < W)
                            ? __ldg(in + ((static_cast<int64_t>(n) * cin + ci) * H + yy) * W + xx)
                            : 0.f;
    }
  for (int o = 0; o < c0; ++o) {
    float acc = 0.f;
    for (int i = 0; i < cin * 9; ++i) acc += ws[o * cin * 9 + i] * win[i];
    out[p * ld + o] = acc;
  }
}

// stem dW partials: split s covers pixels [s*kStemChunk, ...): the chunk's
// upstream gradients (g rows of pitch ld, channels [0, c0)) and its 3x3xcin
// input windows are staged in shared memory, then every weight (o, ci, ky, kx)
// sums its products over the chunk in pixel order -> wpart[s][widx].
__host__ __device__ inline int stem_chunk(int c0, int cin) {  // pixels per split, <= 40 KB staged
  const int c = (40 * 1024) / ((c0 + cin * 9) * 4);
  return c < 16 ? 16 : (c > 128 ? 128 : c);
}
__global__ void k_stem_wgrad(const float* __restrict__ in, int64_t N, int cin, int H, int W,
                             const float* __restrict__ g, int ld, int c0, float* __restrict__ wpart) {
  const int kStemChunk = stem_chunk(c0, cin);
  pdl_enter();
  extern __shared__ float sm[];
  float* gs = sm;                        // [kStemChunk][c0]
  float* xs = sm + kStemChunk * c0;      // [kStemChunk][cin*9]
  const int nt = cin * 9, nw = c0 * nt;
  const int hw = H * W;
  const int64_t M = N * hw;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kStemChunk;
  const int np = static_cast<int>(M - p0 < kStemChunk ? M - p0 : kStemChunk);
  for (int e = threadIdx.x; e < np * c0; e += blockDim.x) {
    const int r = e / c0, o = e - r * c0;
    gs[e] = g[(p0 + r) * ld + o];
  }
  for (int e = threadIdx.x; e < np * nt; e += blockDim.x) {
    const int r = e / nt, t = e - r * nt;
    const int64_t p = p0 + r;
    const int n = static_cast<int>(p / hw);
    const int rem = static_cast<int>(p - static_cast<int64_t>(n) * hw);
    const int ci = t / 9, tap = t - ci * 9;
    const int yy = rem / W + tap / 3 - 1, xx = rem % W + tap % 3 - 1;
    xs[e] = (yy >= 0 && yy < H && xx >= 0 && xx < W)
                ? __ldg(in + ((static_cast<int64_t>(n) * cin + ci) * H + yy) * W + xx)
                : 0.f;
  }
  __syncthreads();
  for (int wi = threadIdx.x; wi < nw; wi += blockDim.x) {
    const int o = wi / nt, t = wi - o * nt;
    float acc = 0.f;
    for (int r = 0; r < np; ++r) acc += gs[r * c0 + o] * xs[r * nt + t];
    wpart[static_cast<int64_t>(blockIdx.x) * nw + wi] = acc;
  }
}

// ---- ImageNet stem (stem == 1; an extension: the reference has only the 3x3 stem) ----
// conv 7x7 stride 2 pad 3 -> BN (batch statistics) -> ReLU -> max-pool 3x3
// stride 2 pad 1, the DenseNet ImageNet stem.  224x224 -> 112x112 -> 56x56, so
// the dense blocks run at 56/28/14/7.  The conv / BN / ReLU
// semantics are the reference's ops (ops.hpp:315-387, :138-243, :248-287) with
// stride 2; the max-pool is restated in oracle/ref_driver.cpp (first maximum
// in (ky, kx) order wins, padding never does).
constexpr int kS7 = 7, kS7Taps = 49;
__host__ __device__ inline int stem7_out(int in) { return (in + 2 * 3 - kS7) / 2 + 1; }  // conv_out_dim
__host__ __device__ inline int pool3_out(int in) { return (in + 2 * 1 - 3) / 2 + 1; }

// y[p][o] (NHWC, pitch c0) = sum_{ci,ky,kx} x[n][ci][2oy-3+ky][2ox-3+kx] w[o][ci][ky][kx],
// the reference's summation order (ops.hpp:321-341).  Thread = two horizontally
// adjacent output pixels x a 32-channel group (blockIdx.y); weights transposed
// in shared memory [tap][c0p], each warp-wide 16-byte weight read is a
// broadcast shared by both pixels (64 FMAs per 8 shared loads).
__global__ void __launch_bounds__(128) k_stem7_conv(const float* __restrict__ in, int64_t N, int cin, int H,
                                                    int W, int Ho, int Wo, const float* __restrict__ w, int c0,
                                                    float* __restrict__ y) {
  pdl_enter();
  extern __shared__ __align__(16) float wsm[];  // [cin*49][c0p]
  const int c0p = (c0 + 31) / 32 * 32, nt = cin * kS7Taps;
  for (int i = threadIdx.x; i < nt * c0p; i += blockDim.x) {
    const int t = i / c0p, o = i - t * c0p;
    wsm[i] = o < c0 ? w[static_cast<int64_t>(o) * nt + t] : 0.f;
  }
  __syncthreads();
  const int wo2 = (Wo + 1) / 2;  // pixel pairs per output row
  const int64_t pair = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pair >= N * Ho * wo2) return;
  const int grp = blockIdx.y;
  const int n = static_cast<int>(pair / (static_cast<int64_t>(Ho) * wo2));
  const int r = static_cast<int>(pair - static_cast<int64_t>(n) * Ho * wo2);
  const int oy = r / wo2, ox = 2 * (r - (r / wo2) * wo2);
  const bool two = ox + 1 < Wo;
  float a0[32], a1[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) a0[j] = a1[j] = 0.f;
  for (int ci = 0; ci < cin; ++ci) {
    const float* xc = in + (static_cast<int64_t>(n) * cin + ci) * H * W;
    for (int ky = 0; ky < kS7; ++ky) {
      const int iy = 2 * oy - 3 + ky;
      if (iy < 0 || iy >= H) continue;
      const float* xr = xc + static_cast<int64_t>(iy) * W;
      for (int kx = 0; kx < kS7; ++kx) {
        const int ix = 2 * ox - 3 + kx;  // pixel 1 reads ix + 2
        const float x0 = (ix >= 0 && ix < W) ? __ldg(xr + ix) : 0.f;
        const float x1 = (ix + 2 >= 0 && ix + 2 < W) ? __ldg(xr + ix + 2) : 0.f;
        const float4* wr = reinterpret_cast<const float4*>(wsm + (ci * kS7Taps + ky * kS7 + kx) * c0p + grp * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 w4 = wr[j];
          a0[4 * j] += x0 * w4.x;
          a0[4 * j + 1] += x0 * w4.y;
          a0[4 * j + 2] += x0 * w4.z;
          a0[4 * j + 3] += x0 * w4.w;
          a1[4 * j] += x1 * w4.x;
          a1[4 * j + 1] += x1 * w4.y;
          a1[4 * j + 2] += x1 * w4.z;
          a1[4 * j + 3] += x1 * w4.w;
        }
      }
    }
  }
  const int64_t p = (static_cast<int64_t>(n) * Ho + oy) * Wo + ox;
  const int nv = c0 - grp * 32 < 32 ? c0 - grp * 32 : 32;
  for (int q = 0; q < (two ? 2 : 1); ++q) {
    const float* a = q ? a1 : a0;
    float* yr = y + (p + q) * c0 + grp * 32;
    if (nv == 32 && (c0 & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        reinterpret_cast<float4*>(yr)[j] = make_float4(a[4 * j], a[4 * j + 1], a[4 * j + 2], a[4 * j + 3]);
    } else {
      for (int j = 0; j < nv; ++j) yr[j] = a[j];
    }
  }
}

// x0[q][c] = max over the 3x3/2 window (pad 1) of relu(bn(y)); arg[q][c] = the
// window tap (ky*3+kx) of the first maximum.  Thread = (q, c), c fastest.
__global__ void k_stem_pool(const float* __restrict__ y, int64_t N, int H1, int W1, int H0, int W0, int c0,
                            const float* __restrict__ mean, const float* __restrict__ var,
                            const float* __restrict__ gamma, const float* __restrict__ beta, float* __restrict__ x0,
                            int ld0, uint8_t* __restrict__ arg) {
  pdl_enter();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= N * H0 * W0 * c0) return;
  const int64_t q = i / c0;
  const int c = static_cast<int>(i - q * c0);
  const int hw0 = H0 * W0;
  const int n = static_cast<int>(q / hw0);
  const int r = static_cast<int>(q - static_cast<int64_t>(n) * hw0);
  const int oy = r / W0, ox = r - (r / W0) * W0;
  const float mu = mean[c], inv = bn_inv(var[c]), ga = gamma[c], be = beta[c];
  float best = 0.f;
  int bt = -1;
  for (int ky = 0; ky < 3; ++ky) {
    const int iy = 2 * oy - 1 + ky;
    if (iy < 0 || iy >= H1) continue;
    for (int kx = 0; kx < 3; ++kx) {
      const int ix = 2 * ox - 1 + kx;
      if (ix < 0 || ix >= W1) continue;
      const float v = fmaxf(bn_ref(y[((static_cast<int64_t>(n) * H1 + iy) * W1 + ix) * c0 + c], mu, inv, ga, be), 0.f);
      if (bt < 0 || v > best) {
        best = v;
        bt = ky * 3 + kx;
      }
    }
  }
  x0[q * ld0 + c] = best;
  arg[q * c0 + c] = static_cast<uint8_t>(bt);
}

// k_stem_pool for c0 % 4 == 0 (and a 16-byte aligned block-input pitch):
// thread = (window q, 4 channels), float4 loads of y, the 3x3 window's nine
// loads issued together; the same first-maximum rule per channel.
__global__ void k_stem_pool4(const float* __restrict__ y, int nq, int H1, int W1, int H0, int W0, int c0,
                             const float* __restrict__ mean, const float* __restrict__ var,
                             const float* __restrict__ gamma, const float* __restrict__ beta,
                             float* __restrict__ x0, int ld0, uint8_t* __restrict__ arg) {
  pdl_enter();
  const int cq = c0 / 4;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq * cq) return;
  const int q = i / cq, c = (i - q * cq) * 4;
  const int hw0 = H0 * W0;
  const int n = q / hw0, r = q - n * hw0;
  const int oy = r / W0, ox = r - (r / W0) * W0;
  const float4 mu = __ldg(reinterpret_cast<const float4*>(mean + c));
  const float4 vr = __ldg(reinterpret_cast<const float4*>(var + c));
  const float4 ga = __ldg(reinterpret_cast<const float4*>(gamma + c));
  const float4 be = __ldg(reinterpret_cast<const float4*>(beta + c));
  const float inv[4] = {bn_inv(vr.x), bn_inv(vr.y), bn_inv(vr.z), bn_inv(vr.w)};
  float4 win[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int iy = 2 * oy - 1 + t / 3, ix = 2 * ox - 1 + t % 3;
    win[t] = (iy >= 0 && iy < H1 && ix >= 0 && ix < W1)
                 ? __ldg(reinterpret_cast<const float4*>(y + ((static_cast<int64_t>(n) * H1 + iy) * W1 + ix) * c0 + c))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float best[4] = {0.f, 0.f, 0.f, 0.f};
  int bt[4] = {-1, -1, -1, -1};
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int iy = 2 * oy - 1 + t / 3, ix = 2 * ox - 1 + t % 3;
    if (iy < 0 || iy >= H1 || ix < 0 || ix >= W1) continue;
    const float w4[4] = {win[t].x, win[t].y, win[t].z, win[t].w};
    const float m4[4] = {mu.x, mu.y, mu.z, mu.w}, g4[4] = {ga.x, ga.y, ga.z, ga.w}, b4[4] = {be.x, be.y, be.z, be.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float v = fmaxf(bn_ref(w4[j], m4[j], inv[j], g4[j], b4[j]), 0.f);
      if (bt[j] < 0 || v > best[j]) {
        best[j] = v;
        bt[j] = t;
      }
    }
  }
  *reinterpret_cast<float4*>(x0 + static_cast<int64_t>(q) * ld0 + c) = make_float4(best[0], best[1], best[2], best[3]);
  *reinterpret_cast<uchar4*>(arg + static_cast<int64_t>(q) * c0 + c) =
      make_uchar4(static_cast<uint8_t>(bt[0]), static_cast<uint8_t>(bt[1]), static_cast<uint8_t>(bt[2]),
                  static_cast<uint8_t>(bt[3]));
}

// Gradient w.r.t. relu(bn(y)) at conv-output pixel p, channel c: the pooled
// gradients g0[q][c] of every window q containing p whose first maximum is p,
// summed in window order (the order the reference-side scatter adds them).
__device__ __forceinline__ float stem_pool_grad_at(int n, int iy, int ix, int c, int H0, int W0, int c0,
                                                   const float* __restrict__ g0, int ld0,
                                                   const uint8_t* __restrict__ arg) {
  // windows q = (oy, ox) with 2*oy-1 <= iy <= 2*oy+1 (and the same in x)
  const int oy1 = min((iy + 1) / 2, H0 - 1), ox1 = min((ix + 1) / 2, W0 - 1);
  float g = 0.f;
  for (int oy = iy / 2; oy <= oy1; ++oy)
    for (int ox = ix / 2; ox <= ox1; ++ox) {
      const int t = (iy - 2 * oy + 1) * 3 + (ix - 2 * ox + 1);
      const int64_t q = (static_cast<int64_t>(n) * H0 + oy) * W0 + ox;
      if (arg[q * c0 + c] == t) g += g0[q * ld0 + c];
    }
  return g;
}
__device__ __forceinline__ float stem_pool_grad(int64_t p, int c, int H1, int W1, int H0, int W0, int c0,
                                                const float* __restrict__ g0, int ld0,
                                                const uint8_t* __restrict__ arg) {
  const int hw1 = H1 * W1;
  const int pi = static_cast<int>(p);  // M1 < 2^31 (dpb_model_create)
  const int n = pi / hw1;
  const int r = pi - n * hw1;
  const int iy = r / W1;
  return stem_pool_grad_at(n, iy, r - iy * W1, c, H0, W0, c0, g0, ld0, arg);
}

// BN backward partial sums of the stem: g = relu'(bn(y)) * stem_pool_grad,
// (sum g, sum g*xhat) over pixel chunk blockIdx.x.  CTA = 32 channel lanes
// (blockIdx.y selects the 32-channel group) x 8 pixel lanes; each warp reads
// one pixel's 32 channels (coalesced); the 8 pixel lanes are folded in fixed
// order (deterministic).
__global__ void __launch_bounds__(256) k_stem_bnb_partials(const float* __restrict__ y, int64_t M1, int H1, int W1,
                                                           int H0, int W0, int c0, const float* __restrict__ mean,
                                                           const float* __restrict__ var,
                                                           const float* __restrict__ gamma,
                                                           const float* __restrict__ beta,
                                                           const float* __restrict__ g0, int ld0,
                                                           const uint8_t* __restrict__ arg, int64_t chunk,
                                                           double2* __restrict__ part) {
  pdl_enter();
  __shared__ double r1[8][33], r2[8][33];
  const int lane = threadIdx.x % 32, pl = threadIdx.x / 32;
  const int c = blockIdx.y * 32 + lane;
  double s1 = 0.0, s2 = 0.0;
  if (c < c0) {
    const float mu = mean[c], inv = bn_inv(var[c]), ga = gamma[c], be = beta[c];
    const int64_t p0 = static_cast<int64_t>(blockIdx.x) * chunk;
    const int64_t p1 = p0 + chunk < M1 ? p0 + chunk : M1;
    for (int64_t p = p0 + pl; p < p1; p += 8) {
      const float x = y[p * c0 + c];
      if (!(bn_ref(x, mu, inv, ga, be) > 0.f)) continue;  // relu_backward (ops.hpp:268-287)
      const float g = stem_pool_grad(p, c, H1, W1, H0, W0, c0, g0, ld0, arg);
      s1 += g;
      s2 += g * ((x - mu) * inv);
    }
  }
  r1[pl][lane] = s1;
  r2[pl][lane] = s2;
  __syncthreads();
  if (pl == 0 && c < c0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < 8; ++i) {
      a += r1[i][lane];
      b += r2[i][lane];
    }
    part[static_cast<int64_t>(blockIdx.x) * c0 + c] = make_double2(a, b);
  }
}

// k_stem_bnb_partials for c0 % 4 == 0 that also stores the masked max-pool
// gradient gm[p][c] = relu'(bn(y)) * stem_pool_grad (dense, pitch c0) for the
// tensor-core dW (StemWgradGemm reads it instead of redoing the gather).
// Thread = (pixel lane, 4 channels): the up-to-four windows' argmax and
// gradient loads are issued together (branch-free), then summed in window
// order (oy, ox ascending: stem_pool_grad_at's order, so g is bit-identical).
// Partials part[cta][c] folded over the pixel lanes in fixed order.
constexpr int kGatherThreads = 256;
__global__ void __launch_bounds__(kGatherThreads) k_stem_bnb_gather(
    const float* __restrict__ y, int64_t M1, int H1, int W1, int H0, int W0, int c0, const float* __restrict__ mean,
    const float* __restrict__ var, const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ g0, int ld0, const uint8_t* __restrict__ arg, int64_t chunk, float* __restrict__ gm,
    double2* __restrict__ part) {
  pdl_enter();
  extern __shared__ double gred[];  // [2][PL][c0]
  const int cq = c0 / 4, PL = kGatherThreads / cq;
  const int lane = threadIdx.x % cq, pl = threadIdx.x / cq;
  const int c = lane * 4;
  double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};
  if (pl < PL) {
    const float4 mu4 = __ldg(reinterpret_cast<const float4*>(mean + c));
    const float4 vr4 = __ldg(reinterpret_cast<const float4*>(var + c));
    const float4 ga4 = __ldg(reinterpret_cast<const float4*>(gamma + c));
    const float4 be4 = __ldg(reinterpret_cast<const float4*>(beta + c));
    const float mu[4] = {mu4.x, mu4.y, mu4.z, mu4.w}, ga[4] = {ga4.x, ga4.y, ga4.z, ga4.w};
    const float be[4] = {be4.x, be4.y, be4.z, be4.w};
    const float inv[4] = {bn_inv(vr4.x), bn_inv(vr4.y), bn_inv(vr4.z), bn_inv(vr4.w)};
    const int hw1 = H1 * W1;
    const int64_t p0 = static_cast<int64_t>(blockIdx.x) * chunk;
    const int64_t p1 = p0 + chunk < M1 ? p0 + chunk : M1;
#pragma unroll 2
    for (int64_t p = p0 + pl; p < p1; p += PL) {
      const int pi = static_cast<int>(p);
      const int n = pi / hw1, r = pi - n * hw1;
      const int iy = r / W1, ix = r - (r / W1) * W1;
      const float4 y4 = __ldg(reinterpret_cast<const float4*>(y + p * c0 + c));
      const int oya = iy / 2, oxa = ix / 2;
      const int oyb = min((iy + 1) / 2, H0 - 1), oxb = min((ix + 1) / 2, W0 - 1);
      uint32_t a[4];
      float4 gv[4];
      int tt[4];
      bool ok[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {  // window order (oya,oxa) (oya,oxb) (oyb,oxa) (oyb,oxb)
        const int oy = w < 2 ? oya : oyb, ox = (w & 1) ? oxb : oxa;
        ok[w] = (w < 2 || oyb != oya) && (!(w & 1) || oxb != oxa);
        tt[w] = (iy - 2 * oy + 1) * 3 + (ix - 2 * ox + 1);
        const int64_t q = (static_cast<int64_t>(n) * H0 + oy) * W0 + ox;
        a[w] = ok[w] ? __ldg(reinterpret_cast<const uint32_t*>(arg + q * c0 + c)) : 0xFFFFFFFFu;
        gv[w] = ok[w] ? __ldg(reinterpret_cast<const float4*>(g0 + q * ld0 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float g[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float v4[4] = {gv[w].x, gv[w].y, gv[w].z, gv[w].w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ok[w] && static_cast<int>((a[w] >> (8 * j)) & 0xFFu) == tt[w]) g[j] += v4[j];
      }
      const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!(bn_ref(yv[j], mu[j], inv[j], ga[j], be[j]) > 0.f)) g[j] = 0.f;  // relu_backward (ops.hpp:268-287)
        s1[j] += g[j];
        s2[j] += g[j] * ((yv[j] - mu[j]) * inv[j]);
      }
      *reinterpret_cast<float4*>(gm + p * c0 + c) = make_float4(g[0], g[1], g[2], g[3]);
    }
  }
  double* r1 = gred;
  double* r2 = gred + PL * c0;
  if (pl < PL) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      r1[pl * c0 + c + j] = s1[j];
      r2[pl * c0 + c + j] = s2[j];
    }
  }
  __syncthreads();
  for (int ch = threadIdx.x; ch < c0; ch += kGatherThreads) {
    double x = 0.0, z = 0.0;
    for (int l = 0; l < PL; ++l) {
      x += r1[l * c0 + ch];
      z += r2[l * c0 + ch];
    }
    part[static_cast<int64_t>(blockIdx.x) * c0 + ch] = make_double2(x, z);
  }
}

// Stem dW partials with the BN-backward apply fused in: a CTA walks output
// tiles of kS7TH x kS7TW pixels (one image each) [tile0, tile1); per tile it
// stages g_y = gamma*inv*(g - mg - xhat*mgx) (ops.hpp:232-241; g = the masked
// max-pool gradient) as [pixel][c0p] and the input window the tile reads
// (cin x (2*TH+5) x (2*TW+5), zero outside the image) in shared memory, then
// thread = a 4-channel x 12-tap register tile of dW[o][t] sums the tile's
// pixels in order.  Partials [cta][c0][cin*49], folded by k_reduce_w1.
constexpr int kS7TH = 8, kS7TW = 16, kS7IH = 2 * kS7TH + 5, kS7IW = 2 * kS7TW + 5, kS7TT = 6;
__host__ __device__ inline int stem7_tiles(int c0, int cin) {  // register tiles = threads
  return ((c0 + 3) / 4) * ((cin * kS7Taps + kS7TT - 1) / kS7TT);
}
__host__ __device__ inline int stem7_wgrad_smem_floats(int c0, int cin) {
  return kS7TH * kS7TW * ((c0 + 3) / 4 * 4) + cin * kS7IH * kS7IW + 6 * c0;
}
__global__ void k_stem7_wgrad(const float* __restrict__ in, int64_t N, int cin, int H, int W, int Ho, int Wo,
                              const float* __restrict__ y, int c0, const float* __restrict__ mean,
                              const float* __restrict__ var, const float* __restrict__ gamma,
                              const float* __restrict__ beta, const float* __restrict__ g0, int ld0, int H0, int W0,
                              const uint8_t* __restrict__ arg, const float* __restrict__ coef, int64_t tiles_per_cta,
                              float* __restrict__ wpart) {
  pdl_enter();
  extern __shared__ __align__(16) float sm7[];
  const int nt = cin * kS7Taps;
  const int c0p = (c0 + 3) / 4 * 4;
  const int ntt = (nt + kS7TT - 1) / kS7TT;
  float* gs = sm7;                               // [TH*TW][c0p]
  float* xs = sm7 + kS7TH * kS7TW * c0p;         // [cin][IH][IW]
  float* tab = xs + cin * kS7IH * kS7IW;         // per channel: mean, inv, gamma, beta, mg, mgx
  for (int c = threadIdx.x; c < c0; c += blockDim.x) {
    tab[6 * c] = mean[c];
    tab[6 * c + 1] = bn_inv(var[c]);
    tab[6 * c + 2] = gamma[c];
    tab[6 * c + 3] = beta[c];
    tab[6 * c + 4] = coef[2 * c];
    tab[6 * c + 5] = coef[2 * c + 1];
  }
  const int tile = threadIdx.x;
  const bool active = tile < stem7_tiles(c0, cin);
  const int og = active ? tile / ntt : 0, tg = active ? tile - og * ntt : 0;
  int tofs[kS7TT];
#pragma unroll
  for (int b = 0; b < kS7TT; ++b) {
    const int t = tg * kS7TT + b;
    const int tc = t < nt ? t : nt - 1;
    const int ci = tc / kS7Taps, tap = tc - ci * kS7Taps;
    tofs[b] = (ci * kS7IH + tap / kS7) * kS7IW + tap % kS7;
  }
  float acc[4][kS7TT];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < kS7TT; ++b) acc[a][b] = 0.f;
  const int tx = (Wo + kS7TW - 1) / kS7TW, ty = (Ho + kS7TH - 1) / kS7TH;
  const int64_t ntiles = N * tx * ty;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * tiles_per_cta;
  const int64_t t1 = t0 + tiles_per_cta < ntiles ? t0 + tiles_per_cta : ntiles;
  for (int64_t ti = t0; ti < t1; ++ti) {
    const int n = static_cast<int>(ti / (tx * ty));
    const int rr = static_cast<int>(ti - static_cast<int64_t>(n) * tx * ty);
    const int oy0 = (rr / tx) * kS7TH, ox0 = (rr - (rr / tx) * tx) * kS7TW;
    __syncthreads();
    for (int e = threadIdx.x; e < kS7TH * kS7TW * c0p; e += blockDim.x) {
      const int pix = e / c0p, c = e - pix * c0p;
      const int oy = oy0 + pix / kS7TW, ox = ox0 + pix % kS7TW;
      float v = 0.f;
      if (c < c0 && oy < Ho && ox < Wo) {
        const int64_t p = (static_cast<int64_t>(n) * Ho + oy) * Wo + ox;
        const float* tc = tab + 6 * c;
        const float mu = tc[0], inv = tc[1], ga = tc[2], be = tc[3];
        const float x = y[p * c0 + c];
        const float g = bn_ref(x, mu, inv, ga, be) > 0.f ? stem_pool_grad_at(n, oy, ox, c, H0, W0, c0, g0, ld0, arg)
                                                         : 0.f;
        v = ga * inv * (g - tc[4] - ((x - mu) * inv) * tc[5]);
      }
      gs[e] = v;
    }
    for (int e = threadIdx.x; e < cin * kS7IH * kS7IW; e += blockDim.x) {
      const int ci = e / (kS7IH * kS7IW), rem = e - ci * kS7IH * kS7IW;
      const int iy = 2 * oy0 - 3 + rem / kS7IW, ix = 2 * ox0 - 3 + rem % kS7IW;
      xs[e] = (iy >= 0 && iy < H && ix >= 0 && ix < W)
                  ? __ldg(in + ((static_cast<int64_t>(n) * cin + ci) * H + iy) * W + ix)
                  : 0.f;
    }
    __syncthreads();
    if (active) {
      for (int py = 0; py < kS7TH; ++py)
        for (int px = 0; px < kS7TW; ++px) {
          const float4 g4 = *reinterpret_cast<const float4*>(gs + (py * kS7TW + px) * c0p + og * 4);
          const float* xb = xs + 2 * py * kS7IW + 2 * px;
          float xv[kS7TT];
#pragma unroll
          for (int b = 0; b < kS7TT; ++b) xv[b] = xb[tofs[b]];
#pragma unroll
          for (int b = 0; b < kS7TT; ++b) {
            acc[0][b] += g4.x * xv[b];
            acc[1][b] += g4.y * xv[b];
            acc[2][b] += g4.z * xv[b];
            acc[3][b] += g4.w * xv[b];
          }
        }
    }
  }
  if (!active) return;
  float* out = wpart + static_cast<int64_t>(blockIdx.x) * c0 * nt;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < kS7TT; ++b) {
      const int o = og * 4 + a, t = tg * kS7TT + b;
      if (o < c0 && t < nt) out[static_cast<int64_t>(o) * nt + t] = acc[a][b];
    }
}

// ---- transition forward: P = avgpool2x2(relu(bn(feat))) --------------------------------
// feat NHWC [N*H*W, C] (pitch C), P [N*Ho*Wo, C]; Ho = H/2, Wo = W/2 (floor,
// ops.hpp:392-402).  bn from the block's batch statistics.
__global__ void k_trans_pool(const float* __restrict__ feat, int ld, int64_t N, int H, int W, int C,
                             const float* __restrict__ mean, const float* __restrict__ var,
                             const float* __restrict__ gamma, const float* __restrict__ beta,
                             float* __restrict__ P) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int Ho = H / 2, Wo = W / 2;
  const float mu = mean[c], inv = bn_inv(var[c]), ga = gamma[c], be = beta[c];
  const int64_t Mq = N * Ho * Wo;
  for (int64_t q = blockIdx.y; q < Mq; q += gridDim.y) {
    const int n = static_cast<int>(q / (Ho * Wo));
    const int r = static_cast<int>(q - static_cast<int64_t>(n) * Ho * Wo);
    const int oy = r / Wo, ox = r - (r / Wo) * Wo;
    const int64_t p = (static_cast<int64_t>(n) * H + 2 * oy) * W + 2 * ox;
    float acc = 0.f;
    acc += fmaxf(bn_ref(feat[p * ld + c], mu, inv, ga, be), 0.f);
    acc += fmaxf(bn_ref(feat[(p + 1) * ld + c], mu, inv, ga, be), 0.f);
    acc += fmaxf(bn_ref(feat[(p + W) * ld + c], mu, inv, ga, be), 0.f);
    acc += fmaxf(bn_ref(feat[(p + W + 1) * ld + c], mu, inv, ga, be), 0.f);
    P[q * C + c] = acc * 0.25f;
  }
}

// k_trans_pool with 16-byte rows (C % 4 == 0, ld % 4 == 0): thread = (pooled
// pixel, 4 channels), the window's four float4 loads issued together.
__global__ void k_trans_pool4(const float* __restrict__ feat, int ld, int64_t Mq, int H, int W, int C,
                              const float* __restrict__ mean, const float* __restrict__ var,
                              const float* __restrict__ gamma, const float* __restrict__ beta,
                              float* __restrict__ P) {
  pdl_enter();
  const int cq = C / 4;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= Mq * cq) return;
  const int64_t q = i / cq;
  const int c = static_cast<int>(i - q * cq) * 4;
  const int Ho = H / 2, Wo = W / 2;
  const int n = static_cast<int>(q / (Ho * Wo));
  const int r = static_cast<int>(q - static_cast<int64_t>(n) * Ho * Wo);
  const int oy = r / Wo, ox = r - (r / Wo) * Wo;
  const int64_t p = (static_cast<int64_t>(n) * H + 2 * oy) * W + 2 * ox;
  const float4 x0 = __ldg(reinterpret_cast<const float4*>(feat + p * ld + c));
  const float4 x1 = __ldg(reinterpret_cast<const float4*>(feat + (p + 1) * ld + c));
  const float4 x2 = __ldg(reinterpret_cast<const float4*>(feat + (p + W) * ld + c));
  const float4 x3 = __ldg(reinterpret_cast<const float4*>(feat + (p + W + 1) * ld + c));
  float m4[4], g4[4], b4[4], inv[4];  // (parameter offsets need not be 16-byte aligned)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    m4[j] = __ldg(mean + c + j);
    inv[j] = bn_inv(__ldg(var + c + j));
    g4[j] = __ldg(gamma + c + j);
    b4[j] = __ldg(beta + c + j);
  }
  const float a0[4] = {x0.x, x0.y, x0.z, x0.w}, a1[4] = {x1.x, x1.y, x1.z, x1.w};
  const float a2[4] = {x2.x, x2.y, x2.z, x2.w}, a3[4] = {x3.x, x3.y, x3.z, x3.w};
  float o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {  // the same sum order as k_trans_pool
    float acc = 0.f;
    acc += fmaxf(bn_ref(a0[j], m4[j], inv[j], g4[j], b4[j]), 0.f);
    acc += fmaxf(bn_ref(a1[j], m4[j], inv[j], g4[j], b4[j]), 0.f);
    acc += fmaxf(bn_ref(a2[j], m4[j], inv[j], g4[j], b4[j]), 0.f);
    acc += fmaxf(bn_ref(a3[j], m4[j], inv[j], g4[j], b4[j]), 0.f);
    o[j] = acc * 0.25f;
  }
  *reinterpret_cast<float4*>(P + q * C + c) = make_float4(o[0], o[1], o[2], o[3]);
}

// running statistics momentum update from a block's batch statistics (biased var)
__global__ void k_running(int C, const float* __restrict__ mean, const float* __restrict__ var,
                          float* __restrict__ run_mean, float* __restrict__ run_var) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  run_mean[c] = (1.f - kMomentum) * run_mean[c] + kMomentum * mean[c];
  run_var[c] = (1.f - kMomentum) * run_var[c] + kMomentum * var[c];
}

// ---- fp32 SIMT GEMM: C[m][n] (+split z) = sum_k A(m,k) B(k,n) ------------------------
// A(m,k) = TA ? A[k*lda + m] : A[m*lda + k];  B(k,n) = TB ? B[n*ldb + k] : B[k*ldb + n].
// Split z covers k in [z*kchunk, ...) and writes Cm + z*M*ldc.  64x64 tiles.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_gemm(int M, int N, int K, const float* __restrict__ A, int lda,
                                              const float* __restrict__ B, int ldb, float* __restrict__ Cm,
                                              int ldc, int kchunk) {
  pdl_enter();
  __shared__ __align__(16) float As[16][64 + 4];
  __shared__ __align__(16) float Bs[16][64 + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int kb = blockIdx.z * kchunk;
  const int ke = kb + kchunk < K ? kb + kchunk : K;
  float acc[4][4] = {};
  for (int k0 = kb; k0 < ke; k0 += 16) {
    // consecutive threads read consecutive addresses: along M (N) for a
    // transposed A (a plain B), along K within a row otherwise
    for (int e = tid; e < 16 * 64; e += 256) {
      const int ka = TA ? e / 64 : e % 16, ma = TA ? e % 64 : e / 16;
      const int kb2 = TB ? e % 16 : e / 64, nb = TB ? e / 16 : e % 64;
      const int gka = k0 + ka, gm = m0 + ma;
      const int gkb = k0 + kb2, gn = n0 + nb;
      As[ka][ma] = (gka < ke && gm < M) ? (TA ? A[static_cast<int64_t>(gka) * lda + gm]
                                              : A[static_cast<int64_t>(gm) * lda + gka])
                                        : 0.f;
      Bs[kb2][nb] = (gkb < ke && gn < N) ? (TB ? B[static_cast<int64_t>(gn) * ldb + gkb]
                                               : B[static_cast<int64_t>(gkb) * ldb + gn])
                                         : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      // 16-byte shared loads (rows of 68 floats: ty*4 / tx*4 offsets stay aligned)
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
  float* out = Cm + static_cast<int64_t>(blockIdx.z) * M * ldc;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gm = m0 + ty * 4 + i, gn = n0 + tx * 4 + j;
      if (gm < M && gn < N) out[static_cast<int64_t>(gm) * ldc + gn] = acc[i][j];
    }
}

// Transition GEMMs of the bf16 path on the tcgen05 engine (tc_gemm_kernel):
// D[M][N] = A . B^T with fp32 operands split into bf16 hi | lo (three MMAs per
// K step, ~16-bit products), fp32 accumulation in TMEM.  A is K-major with row
// pitch lda; B is K-major ([N][K], pitch ldb) or MN-major ([K][N], BMN);
// D has row pitch ldd.  Used for the forward conv (P . W^T) and the pooled-input
// gradient (g_pool . W); the fp32 path keeps k_gemm.
template <int BMN>
struct TransGemm {
  static constexpr int BN = 128;
  static constexpr bool kSplit = true;
  // forward conv (BMN 0): fp16x3 like every forward GEMM (split8_h); the
  // pooled-input gradient (BMN 1) keeps bf16x3 (gradients need bf16's range)
  static constexpr bool kF16 = BMN == 0;
  static constexpr int kAMN = 0, kBMN = BMN;
  static constexpr bool kColSums = false;
  const float* A;
  const float* B;
  float* D;
  int M, N, K, lda, ldb, ldd;

  __device__ int num_kb() const { return (K + tc::kBK - 1) / tc::kBK; }
  __device__ void prologue(uint8_t*) const {}
  // 8 consecutive elements of row `r` (pitch ld, `n` valid), vectorised when aligned
  __device__ static void load8(const float* G, int64_t ld, int r, int rows, int c0, int n, float (&v)[8]) {
    if (r < rows && c0 + 8 <= n && (ld & 3) == 0) {
      const float4* q = reinterpret_cast<const float4*>(G + static_cast<int64_t>(r) * ld + c0);
      const float4 a = __ldg(q), b = __ldg(q + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[i] = (r < rows && c0 + i < n) ? __ldg(G + static_cast<int64_t>(r) * ld + c0 + i) : 0.f;
    }
  }
  __device__ void produce(uint8_t* a_hi, uint8_t* a_lo, uint8_t* b_hi, uint8_t* b_lo, int kb,
                          const uint8_t*) const {
    const int k0 = kb * tc::kBK;
    for (int q = threadIdx.x; q < tc::kBM * tc::kBK / 8; q += tc::kThreads) {
      int row, kc;
      tc::kmajor_coords(q, row, kc);
      float v[8];
      load8(A, lda, blockIdx.x * tc::kBM + row, M, k0 + kc, K, v);
      uint4 h, l;
      if constexpr (kF16) tc::split8_h(v, h, l);
      else tc::split8_fast(v, h, l);
      const uint32_t off = tc::Tile<tc::kBM>::kmajor_chunk(row, kc);
      tc::st_shared16(a_hi, off, h);
      tc::st_shared16(a_lo, off, l);
    }
    for (int q = threadIdx.x; q < BN * tc::kBK / 8; q += tc::kThreads) {
      float v[8];
      uint32_t off;
      if (BMN == 0) {
        int row, kc;
        tc::kmajor_coords(q, row, kc);
        load8(B, ldb, blockIdx.y * BN + row, N, k0 + kc, K, v);
        off = tc::Tile<BN>::kmajor_chunk(row, kc);
      } else {
        int rg, kr;
        tc::mnmajor_coords<BN>(q, rg, kr);
        load8(B, ldb, k0 + kr, K, blockIdx.y * BN + rg, N, v);  // row k of [K][N]
        off = tc::Tile<BN>::mnmajor_chunk(rg, kr);
      }
      uint4 h, l;
      if constexpr (kF16) tc::split8_h(v, h, l);
      else tc::split8_fast(v, h, l);
      tc::st_shared16(b_hi, off, h);
      tc::st_shared16(b_lo, off, l);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&)[8],
                           float (&)[8]) const {
    const int gr = blockIdx.x * tc::kBM + row, gc = blockIdx.y * BN + col0;
    if (gr >= M) return;
    float* d = D + static_cast<int64_t>(gr) * ldd + gc;
    if (gc + 8 <= N && (ldd & 3) == 0) {
      reinterpret_cast<float4*>(d)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(d)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (gc + i < N) d[i] = v[i];
    }
  }
  __device__ void col_sums(int, double, double) const {}
};

// ---- the ImageNet stem on the tcgen05 engine (bf16 path) ---------------------------
// The 7x7 stride-2 pad-3 conv is recast as a stride-1 4x4 conv over the
// space-to-depth image: phase (py, px) of input channel ci is x[ci][2a+py][2b+px],
// and tap (ky, kx) of output pixel (oy, ox) reads phase py = (ky+1)&1 at row
// a = oy + dy with ky = 2*dy + py + 3 (dy in [-2, 1]).  k_stem_s2d writes the
// phases NHWC, zero-padded (2 rows/columns before, 1 after), 16 channel-phases
// per position (cp = (py*2+px)*cin + ci, cin <= 4, the rest zero) as 16-byte
// rows of 8 halves, so every MMA operand chunk of the conv (8 channel-phases of
// one pixel at one (dy, dx)) is ONE 16-byte load: no per-element im2col
// arithmetic, no bounds checks.  Three planes: fp16 hi/lo (the forward's fp16x3
// split, dpb_tc.cuh split8_h) and bf16 (the dW's single bf16 operand).  Tap
// order t' = ((dy+2)*4 + (dx+2))*16 + cp: K = 256, 49*cin of them real.
struct StemS2d {
  int cin, H, W, Ho, Wo;
  __host__ __device__ int rows() const { return Ho + 3; }
  __host__ __device__ int cols() const { return Wo + 3; }
};
__device__ __forceinline__ bool stem_tap_of(int tp, int cin, int& t) {  // t' -> original ci*49 + ky*7 + kx
  const int dd = tp >> 4, cp = tp & 15;
  if (cp >= 4 * cin) return false;
  const int ph = cp / cin, ci = cp - ph * cin;
  const int ky = 2 * (dd >> 2) + (ph >> 1) - 1, kx = 2 * (dd & 3) + (ph & 1) - 1;
  if (ky < 0 || ky >= kS7 || kx < 0 || kx >= kS7) return false;
  t = ci * kS7Taps + ky * kS7 + kx;
  return true;
}
// Blocks [0, img_blocks): thread = one padded position (n, a, b) -> its 16
// channel-phases in the three planes.  Blocks past them: thread = one (o, t')
// of the forward weights in the same tap order (fp16 hi/lo, rows of 256).
__global__ void k_stem_s2d(const float* __restrict__ x, int64_t N, StemS2d g, const float* __restrict__ w, int c0,
                           int wrows, int img_blocks, uint4* __restrict__ xh, uint4* __restrict__ xl,
                           uint4* __restrict__ xb, __half* __restrict__ wh, __half* __restrict__ wl) {
  pdl_enter();
  if (static_cast<int>(blockIdx.x) >= img_blocks) {
    const int i = (blockIdx.x - img_blocks) * blockDim.x + threadIdx.x;
    if (i >= wrows * 256) return;
    const int o = i >> 8, tp = i & 255;
    int t;
    const float v = (o < c0 && stem_tap_of(tp, g.cin, t)) ? w[static_cast<int64_t>(o) * g.cin * kS7Taps + t] : 0.f;
    const __half h = __float2half_rn(v);
    wh[i] = h;
    wl[i] = __float2half_rn(v - __half2float(h));
    return;
  }
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per = static_cast<int64_t>(g.rows()) * g.cols();
  if (i >= N * per) return;
  const int n = static_cast<int>(i / per);
  const int r = static_cast<int>(i - n * per);
  const int a = r / g.cols(), b = r - (r / g.cols()) * g.cols();
  float v[16];
#pragma unroll
  for (int cp = 0; cp < 16; ++cp) {
    v[cp] = 0.f;
    if (cp < 4 * g.cin) {
      const int ph = cp / g.cin, ci = cp - ph * g.cin;
      const int iy = 2 * (a - 2) + (ph >> 1), ix = 2 * (b - 2) + (ph & 1);
      if (iy >= 0 && iy < g.H && ix >= 0 && ix < g.W)
        v[cp] = __ldg(x + ((static_cast<int64_t>(n) * g.cin + ci) * g.H + iy) * g.W + ix);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float e[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = v[8 * h + j];
    uint4 hi, lo;
    tc::split8_h(e, hi, lo);
    xh[2 * i + h] = hi;
    xl[2 * i + h] = lo;
    xb[2 * i + h] = tc::to_bf16x8(e);
  }
}

// y[p][o] = sum_t' s2d(x)[p][t'] W'[o][t'], fp16x3 (hi.hi + hi.lo + lo.hi), fp32
// accumulate; K = 256 in four blocks (kb = dy + 2, the 16 B chunk at K offset
// kc = (dx + 2)*16 + 8*half).  The epilogue stores y (NHWC, pitch c0) and the
// tile's BN column sums (part[tile][c]: k_channel_partials' layout, folded by
// the same finalize).
template <int BN_>
struct StemConvGemm {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = true, kF16 = true, kColSums = true;
  static constexpr int kAMN = 0, kBMN = 0;
  const uint4 *xh, *xl;    // s2d planes (16-byte rows)
  const uint4 *wh, *wl;    // W' [BN][256] halves
  float* y;
  double2* part;
  StemS2d g;
  int c0;
  int64_t M1;

  __device__ int num_kb() const { return 4; }
  __device__ void prologue(uint8_t* aux) const {
    int* base = reinterpret_cast<int*>(aux);  // per tile row: 16-byte row index of (n, oy, ox) at dy = dx = -2
    const int hw = g.Ho * g.Wo;
    for (int row = threadIdx.x; row < tc::kBM; row += tc::kThreads) {
      const int64_t p = static_cast<int64_t>(blockIdx.x) * tc::kBM + row;
      int v = -1;
      if (p < M1) {
        const int pi = static_cast<int>(p);
        const int n = pi / hw, r = pi - n * hw;
        const int oy = r / g.Wo, ox = r - (r / g.Wo) * g.Wo;
        v = ((n * g.rows() + oy) * g.cols() + ox) * 2;
      }
      base[row] = v;
    }
  }
  __device__ void produce(uint8_t* a_hi, uint8_t* a_lo, uint8_t* b_hi, uint8_t* b_lo, int kb,
                          const uint8_t* aux) const {
    const int* base = reinterpret_cast<const int*>(aux);
    const int rowstep = kb * g.cols() * 2;
#pragma unroll
    for (int q = threadIdx.x; q < tc::kBM * tc::kBK / 8; q += tc::kThreads) {
      int row, kc;
      tc::kmajor_coords(q, row, kc);
      const int b0 = base[row];
      uint4 h = make_uint4(0, 0, 0, 0), l = h;
      if (b0 >= 0) {
        const int idx = b0 + rowstep + (kc >> 4) * 2 + ((kc >> 3) & 1);
        h = __ldg(xh + idx);
        l = __ldg(xl + idx);
      }
      const uint32_t off = tc::Tile<tc::kBM>::kmajor_chunk(row, kc);
      tc::st_shared16(a_hi, off, h);
      tc::st_shared16(a_lo, off, l);
    }
#pragma unroll
    for (int q = threadIdx.x; q < BN * tc::kBK / 8; q += tc::kThreads) {
      int row, kc;
      tc::kmajor_coords(q, row, kc);
      const int idx = (row * 256 + kb * tc::kBK + kc) >> 3;
      const uint32_t off = tc::Tile<BN>::kmajor_chunk(row, kc);
      tc::st_shared16(b_hi, off, __ldg(wh + idx));
      tc::st_shared16(b_lo, off, __ldg(wl + idx));
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&s1)[8],
                           float (&s2)[8]) const {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * tc::kBM + row;
    const int nv = p < M1 ? (c0 - col0 < 8 ? c0 - col0 : 8) : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = i < nv;
      s1[i] = ok ? v[i] : 0.f;
      s2[i] = ok ? v[i] * v[i] : 0.f;
    }
    if (nv == 8) {
      float4* dst = reinterpret_cast<float4*>(y + p * c0 + col0);
      dst[0] = make_float4(v[0], v[1], v[2], v[3]);
      dst[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
  __device__ void col_sums(int c, double s1, double s2) const {
    if (c < c0) part[static_cast<int64_t>(blockIdx.x) * c0 + c] = make_double2(s1, s2);
  }
};

// The stem dW: dW[o][t] = sum_p G[p][o] im2col(x)[p][t], K = pixels split over
// blockIdx.z (partials wpart[z][o][t], folded by launch_fold_splits).  A rows =
// the c0 channels of G = gamma*inv*(g - mg - xhat*mgx) (ops.hpp:232-241; g the
// ReLU-masked max-pool gradient k_stem_bnb_gather stored), built in the
// producer from y1 and g (MN-major: 8 channels of one pixel); B rows = the 256
// s2d taps (MN-major: 8 channel-phases of one pixel at one (dy, dx) = one
// 16-byte load of the bf16 plane).  Single bf16 products like the other
// backward GEMMs.  The epilogue maps t' back to (ci, ky, kx).
struct StemWgradGemm {
  static constexpr int BN = 256;
  static constexpr bool kSplit = false, kF16 = false, kColSums = false;
  static constexpr int kAMN = 1, kBMN = 1;
  const uint4* xb;   // bf16 s2d plane
  const float* y1;   // stem conv output [M1][c0]
  const float* gm;   // masked max-pool gradient [M1][c0]
  const float *mean, *var, *gamma, *beta, *coef;
  float* wpart;
  StemS2d g;
  int c0;
  int64_t M1, kchunk;

  __device__ int64_t kbeg() const { return static_cast<int64_t>(blockIdx.z) * kchunk; }
  __device__ int64_t kend() const { return kbeg() + kchunk < M1 ? kbeg() + kchunk : M1; }
  __device__ int num_kb() const { return static_cast<int>((kend() - kbeg() + tc::kBK - 1) / tc::kBK); }
  __device__ void prologue(uint8_t* aux) const {
    float* tab = reinterpret_cast<float*>(aux);  // per channel: mean, inv, gamma, beta, mg, mgx
    for (int c = threadIdx.x; c < c0; c += tc::kThreads) {
      tab[6 * c] = mean[c];
      tab[6 * c + 1] = bn_inv(var[c]);
      tab[6 * c + 2] = gamma[c];
      tab[6 * c + 3] = beta[c];
      tab[6 * c + 4] = coef[2 * c];
      tab[6 * c + 5] = coef[2 * c + 1];
    }
  }
  __device__ void produce(uint8_t* ah, uint8_t*, uint8_t* bh, uint8_t*, int kb, const uint8_t* aux) const {
    const float* tab = reinterpret_cast<const float*>(aux);
    int* base = const_cast<int*>(reinterpret_cast<const int*>(aux + sizeof(float) * 6 * tc::kBM));
    const int64_t pk = kbeg() + static_cast<int64_t>(kb) * tc::kBK, pe = kend();
    if (threadIdx.x < tc::kBK) {  // this K block's pixels -> s2d row index (the engine's barrier
      const int64_t p = pk + threadIdx.x;  // after produce(kb - 1) ordered the previous readers)
      int v = -1;
      if (p < pe) {
        const int hw = g.Ho * g.Wo, pi = static_cast<int>(p);
        const int n = pi / hw, r = pi - n * hw;
        const int oy = r / g.Wo, ox = r - (r / g.Wo) * g.Wo;
        v = ((n * g.rows() + oy) * g.cols() + ox) * 2;
      }
      base[threadIdx.x] = v;
    }
    // A: 8 channels of G at one pixel (rows >= c0 stay zero after each stage's first fill)
#pragma unroll
    for (int q = threadIdx.x; q < tc::kBM * tc::kBK / 8; q += tc::kThreads) {
      int rg, kr;
      tc::mnmajor_coords<tc::kBM>(q, rg, kr);
      if (rg >= c0 && kb >= 2) continue;
      const int64_t p = pk + kr;
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
      if (p < pe && rg < c0) {
        float gv[8], yv[8];
        tc::load8(gm + p * c0 + rg, 8, true, gv);
        tc::load8(y1 + p * c0 + rg, 8, true, yv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float* t = tab + 6 * (rg + i);
          const float mu = t[0], inv = t[1], ga = t[2];
          v[i] = ga * inv * (gv[i] - t[4] - ((yv[i] - mu) * inv) * t[5]);
        }
      }
      tc::st_shared16(ah, tc::Tile<tc::kBM>::mnmajor_chunk(rg, kr), tc::to_bf16x8(v));
    }
    __syncthreads();  // the pixel table
    // B: 8 channel-phases at one (pixel, dy, dx): one 16-byte load
#pragma unroll 4
    for (int q = threadIdx.x; q < BN * tc::kBK / 8; q += tc::kThreads) {
      int rg, kr;
      tc::mnmajor_coords<BN>(q, rg, kr);
      const int b0 = base[kr];
      const int dd = rg >> 4;
      const uint4 v = b0 >= 0 ? __ldg(xb + b0 + ((dd >> 2) * g.cols() + (dd & 3)) * 2 + ((rg >> 3) & 1))
                              : make_uint4(0, 0, 0, 0);
      tc::st_shared16(bh, tc::Tile<BN>::mnmajor_chunk(rg, kr), v);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&)[8],
                           float (&)[8]) const {
    if (row >= c0) return;
    const int nt = g.cin * kS7Taps;
    float* dst = wpart + (static_cast<int64_t>(blockIdx.z) * c0 + row) * nt;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int t;
      if (stem_tap_of(col0 + i, g.cin, t)) dst[t] = v[i];
    }
  }
  __device__ void col_sums(int, double, double) const {}
};

// Transition dW partials on the tcgen05 engine (bf16 path): wpart[z][o][c] =
// sum over pixel chunk z of g_pool[p][o] P[p][c] (graph.hpp transition conv
// backward; the fp32 path keeps k_gemm<true, false>).  A rows = the cout
// output channels, B rows = the C input channels, both MN-major (8 channels of
// one pixel per 16-byte chunk), K = pooled pixels; single bf16 products like
// the dense layers' dW GEMMs.
struct TransWgradGemm {
  static constexpr int BN = 128;
  static constexpr bool kSplit = false, kF16 = false, kColSums = false;
  static constexpr int kAMN = 1, kBMN = 1;
  const float* G;  // [Mq][ldg] pooled-output gradient (channels [0, cout))
  const float* P;  // [Mq][C] pooled activations
  float* wpart;
  int cout, C, ldg;
  int64_t Mq, kchunk;

  __device__ int64_t kbeg() const { return static_cast<int64_t>(blockIdx.z) * kchunk; }
  __device__ int64_t kend() const { return kbeg() + kchunk < Mq ? kbeg() + kchunk : Mq; }
  __device__ int num_kb() const { return static_cast<int>((kend() - kbeg() + tc::kBK - 1) / tc::kBK); }
  __device__ void prologue(uint8_t*) const {}
  __device__ void produce(uint8_t* ah, uint8_t*, uint8_t* bh, uint8_t*, int kb, const uint8_t*) const {
    const int64_t pk = kbeg() + static_cast<int64_t>(kb) * tc::kBK, pe = kend();
    const int m0 = blockIdx.x * tc::kBM, n0 = blockIdx.y * BN;
#pragma unroll
    for (int q = threadIdx.x; q < tc::kBM * tc::kBK / 8; q += tc::kThreads) {
      int rg, kr;
      tc::mnmajor_coords<tc::kBM>(q, rg, kr);
      const int64_t p = pk + kr;
      float v[8];
      if (p < pe && m0 + rg < cout) tc::load8(G + p * ldg + m0 + rg, cout - m0 - rg, (ldg & 3) == 0, v);
      else tc::zero8(v);
      tc::st_shared16(ah, tc::Tile<tc::kBM>::mnmajor_chunk(rg, kr), tc::to_bf16x8(v));
    }
#pragma unroll
    for (int q = threadIdx.x; q < BN * tc::kBK / 8; q += tc::kThreads) {
      int rg, kr;
      tc::mnmajor_coords<BN>(q, rg, kr);
      const int64_t p = pk + kr;
      float v[8];
      if (p < pe && n0 + rg < C) tc::load8(P + p * C + n0 + rg, C - n0 - rg, (C & 3) == 0, v);
      else tc::zero8(v);
      tc::st_shared16(bh, tc::Tile<BN>::mnmajor_chunk(rg, kr), tc::to_bf16x8(v));
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&)[8],
                           float (&)[8]) const {
    const int o = blockIdx.x * tc::kBM + row, c = blockIdx.y * BN + col0;
    if (o < cout && c < C)
      tc::store8(wpart + (static_cast<int64_t>(blockIdx.z) * cout + o) * C + c, C - c, (C & 3) == 0, v);
  }
  __device__ void col_sums(int, double, double) const {}
};

template <int BMN>
void trans_gemm(cudaStream_t st, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                float* D, int ldd) {
  using Op = TransGemm<BMN>;
  const Op op{A, B, D, M, N, K, lda, ldb, ldd};
  launch(tc::tc_gemm_kernel<Op>, dim3((M + tc::kBM - 1) / tc::kBM, (N + Op::BN - 1) / Op::BN), tc::kThreads,
         tc::stage_bytes<Op>(), st, op);
}

// ---- head forward: gap[n][c] = mean_hw relu(bn(feat)) ---------------------------------
__global__ void k_head_gap(const float* __restrict__ feat, int ld, int64_t N, int HW, int C,
                           const float* __restrict__ mean, const float* __restrict__ var,
                           const float* __restrict__ gamma, const float* __restrict__ beta,
                           float* __restrict__ gap) {
  pdl_enter();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= N * C) return;
  const int c = static_cast<int>(i % C);
  const int64_t n = i / C;
  const float inv = bn_inv(var[c]);
  float acc = 0.f;
  for (int p = 0; p < HW; ++p)
    acc += fmaxf(bn_ref(feat[(n * HW + p) * ld + c], mean[c], inv, gamma[c], beta[c]), 0.f);
  gap[i] = acc * (1.f / static_cast<float>(HW));
}

// logits = gap . W^T + b; softmax cross entropy (ops.hpp:528-559): one CTA per
// sample; per-sample loss (mean taken by k_loss_mean), g_logits = (p - onehot)/N.
// logits[n][o] = b[o] + sum_c W[o][c] gap[n][c] (linear_forward, ops.hpp:474-485):
// one warp per (class o, group of kLogitRows samples); lanes stride over C
// (coalesced W row, read once per group), fixed butterfly per sample.
constexpr int kLogitRows = 8;
__global__ void k_head_logits(const float* __restrict__ gap, int64_t N, int C, const float* __restrict__ Wl,
                              const float* __restrict__ bl, int classes, float* __restrict__ logits) {
  pdl_enter();
  const int lane = threadIdx.x % 32;
  const int64_t wid = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int64_t groups = (N + kLogitRows - 1) / kLogitRows;
  if (wid >= groups * classes) return;
  const int o = static_cast<int>(wid % classes);
  const int64_t n0 = (wid / classes) * kLogitRows;
  float acc[kLogitRows];
#pragma unroll
  for (int r = 0; r < kLogitRows; ++r) acc[r] = 0.f;
  const float* wr = Wl + static_cast<int64_t>(o) * C;
  for (int c = lane; c < C; c += 32) {
    const float wv = wr[c];
#pragma unroll
    for (int r = 0; r < kLogitRows; ++r)
      if (n0 + r < N) acc[r] += wv * gap[(n0 + r) * C + c];
  }
#pragma unroll
  for (int r = 0; r < kLogitRows; ++r) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
    if (lane == 0 && n0 + r < N) logits[(n0 + r) * classes + o] = bl[o] + acc[r];
  }
}

__global__ void k_head_loss(const float* __restrict__ gap, int64_t N, int C, const float* __restrict__ Wl,
                            const float* __restrict__ bl, int classes, const int32_t* __restrict__ labels,
                            float* __restrict__ logits, float* __restrict__ g_logits,
                            float* __restrict__ loss_n, int* __restrict__ bad_label) {
  pdl_enter();
  __shared__ float red[256];
  const int64_t n = blockIdx.x;
  const float* lg = logits + n * classes;  // written by k_head_logits
  // max and sum of exp, fixed-order tree over the CTA
  float mx = -INFINITY;
  for (int o = threadIdx.x; o < classes; o += blockDim.x) mx = fmaxf(mx, lg[o]);
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  float sm = 0.f;
  for (int o = threadIdx.x; o < classes; o += blockDim.x) sm += expf(lg[o] - mx);
  red[threadIdx.x] = sm;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const float log_sum = logf(red[0]) + mx;
  const int label = labels[n];
  if (label < 0 || label >= classes) {
    // LabelError (ops.hpp softmax_xent): flagged for dpb_model_sync, and the
    // sample's loss and logit gradients are NaN so a step that ignores the
    // flag cannot silently train on stale values
    for (int o = threadIdx.x; o < classes; o += blockDim.x) g_logits[n * classes + o] = __int_as_float(0x7fc00000);
    if (threadIdx.x == 0) {
      *bad_label = 1;
      loss_n[n] = __int_as_float(0x7fc00000);
    }
    return;
  }
  for (int o = threadIdx.x; o < classes; o += blockDim.x) {
    const float p = expf(lg[o] - log_sum);
    g_logits[n * classes + o] = (p - (o == label ? 1.f : 0.f)) / static_cast<float>(N);
  }
  if (threadIdx.x == 0) loss_n[n] = log_sum - lg[label];
}

__global__ void k_loss_mean(const float* __restrict__ loss_n, int64_t N, float* __restrict__ loss) {
  pdl_enter();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float s = 0.f;
  for (int64_t i = 0; i < N; ++i) s += loss_n[i];
  *loss = s / static_cast<float>(N);
}

// linear backward (ops.hpp:487-523): g_gap = g_logits . W, dW = g_logits^T . gap,
// db = sum_n g_logits.  One thread per output element, fixed-order sums.
__global__ void k_head_linear_bwd(const float* __restrict__ g_logits, const float* __restrict__ gap,
                                  const float* __restrict__ Wl, int64_t N, int C, int classes,
                                  float* __restrict__ g_gap, float* __restrict__ dW, float* __restrict__ db) {
  pdl_enter();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n_gg = N * C, n_dw = static_cast<int64_t>(classes) * C;
  if (i < n_gg) {
    const int64_t n = i / C;
    const int c = static_cast<int>(i % C);
    float acc = 0.f;
    for (int o = 0; o < classes; ++o) acc += Wl[static_cast<int64_t>(o) * C + c] * g_logits[n * classes + o];
    g_gap[i] = acc;
  } else if (i < n_gg + n_dw) {
    const int64_t j = i - n_gg;
    const int o = static_cast<int>(j / C), c = static_cast<int>(j % C);
    float acc = 0.f;
    for (int64_t n = 0; n < N; ++n) acc += g_logits[n * classes + o] * gap[n * C + c];
    dW[j] = acc;
  } else if (i < n_gg + n_dw + classes) {
    const int o = static_cast<int>(i - n_gg - n_dw);
    float acc = 0.f;
    for (int64_t n = 0; n < N; ++n) acc += g_logits[n * classes + o];
    db[o] = acc;
  }
}

// ---- BN backward of a transition / the head -------------------------------------------
// Upstream gradient of act = relu(bn(x)) at pixel p, channel c:
//   head:        g_gap[n][c] / HW
//   transition:  g_P[q(p)][c] / 4 inside the pooled windows, 0 outside
struct HeadGrad {
  const float* g_gap;
  int HW, C;
  __device__ float operator()(int64_t p, int c) const {
    return g_gap[static_cast<int64_t>(static_cast<int>(p / HW)) * C + c] * (1.f / static_cast<float>(HW));
  }
};
struct PoolGrad {
  const float* g_P;  // [N*Ho*Wo, C]
  int H, W, C;
  __device__ float operator()(int64_t p, int c) const {
    const int Ho = H / 2, Wo = W / 2, hw = H * W;
    const int n = static_cast<int>(p / hw);
    const int r = static_cast<int>(p - static_cast<int64_t>(n) * hw);
    const int y = r / W, x = r - (r / W) * W;
    if (y >= 2 * Ho || x >= 2 * Wo) return 0.f;
    return g_P[((static_cast<int64_t>(n) * Ho + y / 2) * Wo + x / 2) * C + c] * 0.25f;
  }
};

// per-split partial sums (sum g, sum g*xhat) of g = relu'(act) * upstream, over
// pixels [s*chunk, ...): thread = channel, fixed pixel order -> part[s][c]
template <class G>
__global__ void k_bnb_partials(const float* __restrict__ feat, int ld, int64_t M, int C, const float* __restrict__ mean,
                               const float* __restrict__ var, const float* __restrict__ gamma,
                               const float* __restrict__ beta, G up, int64_t chunk, double2* __restrict__ part) {
  pdl_enter();
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const float inv = bn_inv(var[c]);
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t p1 = p0 + chunk < M ? p0 + chunk : M;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
  for (int64_t p = p0; p < p1; ++p) {
    const float x = feat[p * ld + c];
    if (!(bn_ref(x, mean[c], inv, gamma[c], beta[c]) > 0.f)) continue;  // relu_backward
    const float g = up(p, c);
    s1 += g;
    s2 += g * ((x - mean[c]) * inv);
  }
  part[static_cast<int64_t>(blockIdx.x) * C + c] = make_double2(s1, s2);
}

// out[p][c] = (gamma*inv) * (g - mg - xhat*mgx)  (written, ops.hpp:232-241);
// thread = channel (coalesced), grid.y strides over pixels
template <class G>
__global__ void k_bnb_apply(const float* __restrict__ feat, int ld, int64_t M, int C, const float* __restrict__ mean,
                            const float* __restrict__ var, const float* __restrict__ gamma,
                            const float* __restrict__ beta, G up, const float* __restrict__ coef,
                            float* __restrict__ out, int ldo) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const float mu = mean[c], inv = bn_inv(var[c]), ga = gamma[c], be = beta[c];
  const float gi = ga * inv, mg = coef[2 * c], mgx = coef[2 * c + 1];
  for (int64_t p = blockIdx.y; p < M; p += gridDim.y) {
    const float x = feat[p * ld + c];
    const float g = bn_ref(x, mu, inv, ga, be) > 0.f ? up(p, c) : 0.f;
    const float xh = (x - mu) * inv;
    out[p * ldo + c] = gi * (g - mg - xh * mgx);
  }
}

// Transition BN backward for even H, W: every pixel lies in exactly one 2x2
// pooling window, so both passes walk the pooled pixels q (n, oy, ox) of a
// contiguous range with stepped indices (no divisions), loading g_P once per
// window.  Thread = channel (coalesced); partial rows = ranges (fixed order).
__device__ __forceinline__ void pool_walk_start(int64_t q, int Ho, int Wo, int64_t& n, int& oy, int& ox) {
  n = q / (static_cast<int64_t>(Ho) * Wo);
  const int r = static_cast<int>(q - n * Ho * Wo);
  oy = r / Wo;
  ox = r - oy * Wo;
}

__global__ void k_pool_bnb_partials(const float* __restrict__ feat, int ld, int H, int W, int C,
                                    const float* __restrict__ mean, const float* __restrict__ var,
                                    const float* __restrict__ gamma, const float* __restrict__ beta,
                                    const float* __restrict__ g_P, int64_t Mq, int64_t chunk,
                                    double2* __restrict__ part) {
  pdl_enter();
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const float mu = mean[c], inv = bn_inv(var[c]), ga = gamma[c], be = beta[c];
  const int Ho = H / 2, Wo = W / 2;
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t q1 = q0 + chunk < Mq ? q0 + chunk : Mq;
  int64_t n;
  int oy, ox;
  pool_walk_start(q0, Ho, Wo, n, oy, ox);
  double s1 = 0.0, s2 = 0.0;
  for (int64_t q = q0; q < q1; ++q) {
    const float g = g_P[q * C + c] * 0.25f;
    const int64_t p = (n * H + 2 * oy) * W + 2 * ox;
    const int64_t ps[4] = {p, p + 1, p + W, p + W + 1};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float x = feat[ps[t] * ld + c];
      if (bn_ref(x, mu, inv, ga, be) > 0.f) {
        s1 += g;
        s2 += g * ((x - mu) * inv);
      }
    }
    if (++ox == Wo) {
      ox = 0;
      if (++oy == Ho) {
        oy = 0;
        ++n;
      }
    }
  }
  part[static_cast<int64_t>(blockIdx.x) * C + c] = make_double2(s1, s2);
}

__global__ void k_pool_bnb_apply(const float* __restrict__ feat, int ld, int H, int W, int C,
                                 const float* __restrict__ mean, const float* __restrict__ var,
                                 const float* __restrict__ gamma, const float* __restrict__ beta,
                                 const float* __restrict__ g_P, int64_t Mq, int64_t chunk,
                                 const float* __restrict__ coef, float* __restrict__ out, int ldo) {
  pdl_enter();
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const float mu = mean[c], inv = bn_inv(var[c]), ga = gamma[c], be = beta[c];
  const float gi = ga * inv, mg = coef[2 * c], mgx = coef[2 * c + 1];
  const int Ho = H / 2, Wo = W / 2;
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t q1 = q0 + chunk < Mq ? q0 + chunk : Mq;
  int64_t n;
  int oy, ox;
  pool_walk_start(q0, Ho, Wo, n, oy, ox);
  for (int64_t q = q0; q < q1; ++q) {
    const float g = g_P[q * C + c] * 0.25f;
    const int64_t p = (n * H + 2 * oy) * W + 2 * ox;
    const int64_t ps[4] = {p, p + 1, p + W, p + W + 1};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float x = feat[ps[t] * ld + c];
      const float gg = bn_ref(x, mu, inv, ga, be) > 0.f ? g : 0.f;
      out[ps[t] * ldo + c] = gi * (gg - mg - ((x - mu) * inv) * mgx);
    }
    if (++ox == Wo) {
      ox = 0;
      if (++oy == Ho) {
        oy = 0;
        ++n;
      }
    }
  }
}

unsigned blocks_of(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

// ---- the network plan ------------------------------------------------------------------
struct ModelBlock {
  Block* blk = nullptr;
  int64_t M = 0;
  int h = 0, w = 0, c0 = 0, m = 0, C = 0;
  int Cp = 0;            // padded row pitch of the block's features and of acc
  int64_t poff = 0, pelems = 0, roff = 0, relems = 0;
  float* x = nullptr;    // NHWC [M, c0] block input
  float* acc = nullptr;  // NHWC [M, C] block output gradient (in/out)
};
struct ModelTrans {
  int C = 0, cout = 0;  // in (block C) / out channels
  int64_t Mq = 0;       // pooled pixels
  int64_t gamma = 0, beta = 0, w = 0, run = 0;  // offsets
  float* P = nullptr;   // [Mq, C] pooled activations
  float* gP = nullptr;  // [Mq, C]
  float* wpart = nullptr;  // split-K partials of its dW (side stream)
};

}  // namespace dpb

struct dpb_model {
  dpb_model_desc d{};
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;             // transition dW GEMMs + folds (gradient-only work)
  std::vector<cudaEvent_t> ev;             // per transition: fork; plus one join
  std::vector<dpb::ModelBlock> blocks;
  std::vector<dpb::ModelTrans> trans;
  int64_t params = 0, running = 0;
  int64_t head_gamma = 0, head_beta = 0, head_w = 0, head_b = 0, head_run = 0;
  void* mem = nullptr;
  float *gap = nullptr, *logits = nullptr, *g_logits = nullptr, *g_gap = nullptr, *loss_n = nullptr;
  float* wpart = nullptr;
  double2* part = nullptr;
  float* coef = nullptr;
  int* bad_label = nullptr;
  int64_t wpart_elems = 0, part_rows = 0;
  // ImageNet stem (d.stem == 1): conv output y1 [M1, c0], max-pool taps,
  // BN partials / statistics, parameter offsets
  int H1 = 0, W1 = 0;
  int64_t M1 = 0, P1 = 0;
  int64_t stem_w = 0, stem_gamma = 0, stem_beta = 0;
  float* y1 = nullptr;
  uint8_t* arg = nullptr;
  double2* spart = nullptr;
  // the tensor-core stem (bf16 path): space-to-depth image planes (fp16 hi/lo,
  // bf16), forward weights in s2d tap order, masked max-pool gradient
  bool tc_stem = false;
  dpb::StemS2d s2d{};
  uint4 *xh = nullptr, *xl = nullptr, *xb = nullptr;
  __half *wh = nullptr, *wl = nullptr;
  float* gm = nullptr;
  float* sstat = nullptr;  // mean[c0] | var[c0]
  // CUDA graph of the whole step, replayed while the step's buffers stay the same
  cudaGraphExec_t graph = nullptr;
  const void* graph_key[6] = {};
  int64_t graph_kernels = 0;      // kernel nodes of the captured step
  int64_t eager_launches = 0;     // launches of the last eager step
  dpb::DeviceTracker tracker;     // every device allocation of the model
  // data parallelism: per-bucket gradient allreduce on `cstream` (dpb_comm.cu)
  dpb::Comm* comm = nullptr;
  cudaStream_t cstream = nullptr;
  std::vector<cudaEvent_t> ev_tdone;   // per transition: its dW (side stream) written
  std::vector<cudaEvent_t> ev_bucket;  // per block bucket: its gradients written (main)
  cudaEvent_t ev_cjoin = nullptr;      // every bucket reduced
  // the step's last read of its input images and labels (an external event
  // node inside the captured graph): dpb_model_wait_input lets the caller's
  // copy stream bring in the next batch while the rest of the step runs
  cudaEvent_t ev_input = nullptr;
  int64_t mem_tags[6] = {};       // bytes of m->mem per arena tag
};

namespace dpb {
namespace {

constexpr int kSplitsMax = 148;      // split-K of the transition dW GEMM (upper bound)

// Split-K of the transition dW GEMM [cout x C] over its Mq pooled pixels: as
// many splits as bring its 64x64 output tiles to ~4 waves (at least 64 pixels
// per split) — wide transitions have thousands of tiles and need no split,
// and their partials (splits x cout x C fp32) would otherwise run to GBs.
int trans_dw_splits(const ModelTrans& t, int64_t& chunk) {
  const int64_t tiles = ((t.cout + 63) / 64) * ((t.C + 63) / 64);
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>(kSplitsMax, (4 * 148 + tiles - 1) / tiles));
  chunk = std::max<int64_t>(64, (t.Mq + want - 1) / want);
  return static_cast<int>((t.Mq + chunk - 1) / chunk);
}
constexpr int kStem7Splits = 296;    // CTAs (tile ranges) of the 7x7 stem dW (888 measured slower)
constexpr int kRowSplitsMax = 2048;  // pixel chunks of the BN-backward sums and the stem dW

int model_geometry(const dpb_model_desc* d, dpb_model* m) {
  if (d == nullptr) return fail(DPB_CONFIG_ERROR, "null model descriptor");
  if (d->nblocks < 1 || d->nblocks > 8) return fail(DPB_CONFIG_ERROR, "nblocks must be in [1, 8]");
  if (d->k < 1 || d->c0 < 1 || d->classes < 1 || d->in_c < 1 || d->batch < 1)
    return fail(DPB_SHAPE_ERROR, "invalid network geometry");
  if (d->in_c > 4) return fail(DPB_CONFIG_ERROR, "the stem supports at most 4 input channels");
  if (d->stem != 0 && d->stem != 1) return fail(DPB_CONFIG_ERROR, "stem must be 0 (3x3) or 1 (ImageNet 7x7/2)");
  if (!(d->compression > 0.0) || d->compression > 1.0)
    return fail(DPB_CONFIG_ERROR, "compression must be in (0, 1]");
  if (d->dtype != DPB_FP32 && d->dtype != DPB_BF16) return fail(DPB_CONFIG_ERROR, "dtype");
  int h = d->in_h, w = d->in_w, c = d->c0;
  int64_t po = static_cast<int64_t>(d->c0) * d->in_c * 9, ro = 0;
  m->stem_w = 0;
  if (d->stem == 1) {
    // stem.conv.w [c0][in_c][7][7], stem.bn.gamma [c0], stem.bn.beta [c0];
    // running statistics of the stem BN first
    m->H1 = stem7_out(d->in_h);
    m->W1 = stem7_out(d->in_w);
    if (m->H1 < 1 || m->W1 < 1) return fail(DPB_SHAPE_ERROR, "stem conv output collapses to zero size");
    h = pool3_out(m->H1);
    w = pool3_out(m->W1);
    m->M1 = d->batch * m->H1 * m->W1;
    if (m->M1 * d->c0 >= (int64_t{1} << 31)) return fail(DPB_CONFIG_ERROR, "ImageNet stem output beyond 2^31 elements");
    m->P1 = (m->M1 + 127) / 128;
    m->stem_gamma = static_cast<int64_t>(d->c0) * d->in_c * kS7Taps;
    m->stem_beta = m->stem_gamma + d->c0;
    po = m->stem_beta + d->c0;
    ro = 2 * d->c0;
  }
  const int bk = 4 * d->k;
  m->blocks.clear();
  m->trans.clear();
  for (int b = 0; b < d->nblocks; ++b) {
    if (d->blocks[b] < 1) return fail(DPB_SHAPE_ERROR, "every block needs >= 1 layer");
    if (h < 1 || w < 1) return fail(DPB_SHAPE_ERROR, "spatial size collapses to zero");
    ModelBlock mb;
    mb.M = d->batch * h * w;
    mb.h = h;
    mb.w = w;
    mb.c0 = c;
    mb.m = d->blocks[b];
    mb.C = c + mb.m * d->k;
    mb.Cp = (mb.C + 3) / 4 * 4;
    dpb_block_desc bd{d->batch, h, w, c, mb.m, d->k, bk, d->dtype, DPB_NHWC};
    dpb_arena_sizes sz{};
    int rc = validate(&bd);
    if (rc) return rc;
    plan_arena(bd, &sz);
    mb.poff = po;
    mb.pelems = sz.param_elems;
    mb.roff = ro;
    mb.relems = sz.stat_elems;
    po += sz.param_elems;
    ro += sz.stat_elems;
    m->blocks.push_back(mb);
    if (b + 1 < d->nblocks) {
      ModelTrans t;
      t.C = mb.C;
      t.cout = static_cast<int>(std::floor(d->compression * mb.C));  // densenet.hpp:118
      if (t.cout < 1) return fail(DPB_CONFIG_ERROR, "compression collapses channels to 0");
      if (h < 2 || w < 2) return fail(DPB_SHAPE_ERROR, "avgpool output collapses to zero size");
      t.Mq = d->batch * (h / 2) * (w / 2);
      t.gamma = po;
      t.beta = po + t.C;
      t.w = po + 2 * t.C;
      po += 2 * t.C + static_cast<int64_t>(t.cout) * t.C;
      t.run = ro;
      ro += 2 * t.C;
      m->trans.push_back(t);
      c = t.cout;
      h /= 2;
      w /= 2;
    }
  }
  const int C = m->blocks.back().C;
  m->head_gamma = po;
  m->head_beta = po + C;
  m->head_w = po + 2 * C;
  m->head_b = m->head_w + static_cast<int64_t>(d->classes) * C;
  po = m->head_b + d->classes;
  m->head_run = ro;
  ro += 2 * C;
  m->params = po;
  m->running = ro;
  return DPB_OK;
}

}  // namespace
}  // namespace dpb

using namespace dpb;

extern "C" {

DPB_API int dpb_model_sizes(const dpb_model_desc* desc, int64_t* param_elems, int64_t* running_elems) {
  dpb_model m;
  const int rc = model_geometry(desc, &m);
  if (rc) return rc;
  if (param_elems) *param_elems = m.params;
  if (running_elems) *running_elems = m.running;
  return DPB_OK;
}

// GraphPlan<T>::build's parameter init, replayed draw for draw (graph.hpp:
// 351-390 make_bn / make_conv, :405-600 registration order, rng.hpp:14-50):
// one Rng(seed) stream; conv weights float(normal() * sqrt(2 / fan_in)) in
// (oc, ic, ky, kx) order, BN gamma 1 / beta 0, classifier float(sqrt(1 / C) *
// normal()), bias 0.  The ImageNet stem (stem 1, not in the reference) draws
// its 7x7 weights in the same position the reference draws its 3x3 stem.
namespace {
struct HostRng {  // Rng (rng.hpp): mt19937_64, 53-bit uniform, Box-Muller with a spare
  std::mt19937_64 eng;
  bool have = false;
  double spare = 0.0;
  explicit HostRng(uint64_t seed) : eng(seed) {}
  double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    double u1 = uniform();
    const double u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * 3.14159265358979323846 * u2;
    spare = r * std::sin(th);
    have = true;
    return r * std::cos(th);
  }
};
}  // namespace

DPB_API int dpb_model_init_params(const dpb_model_desc* desc, uint64_t seed, float* host_params) {
  if (host_params == nullptr) return fail(DPB_CONFIG_ERROR, "null parameter buffer");
  dpb_model m;
  const int rc = model_geometry(desc, &m);
  if (rc) return rc;
  HostRng rng(seed);
  float* p = host_params;
  auto conv = [&](int64_t out_c, int64_t in_c, int kk) {  // make_conv
    const double stddev = std::sqrt(2.0 / (static_cast<double>(in_c) * kk * kk));
    const int64_t n = out_c * in_c * kk * kk;
    for (int64_t i = 0; i < n; ++i) *p++ = static_cast<float>(rng.normal() * stddev);
  };
  auto bn = [&](int64_t c) {  // make_bn: gamma 1, beta 0
    for (int64_t i = 0; i < c; ++i) *p++ = 1.f;
    for (int64_t i = 0; i < c; ++i) *p++ = 0.f;
  };
  const int bk = 4 * desc->k;
  if (desc->stem == 1) {
    conv(desc->c0, desc->in_c, kS7);
    bn(desc->c0);
  } else {
    conv(desc->c0, desc->in_c, 3);
  }
  for (size_t b = 0; b < m.blocks.size(); ++b) {
    const ModelBlock& mb = m.blocks[b];
    for (int l = 0; l < mb.m; ++l) {
      const int64_t c = mb.c0 + static_cast<int64_t>(l) * desc->k;
      bn(c);
      conv(bk, c, 1);
      bn(bk);
      conv(desc->k, bk, 3);
    }
    if (b + 1 < m.blocks.size()) {
      bn(m.trans[b].C);
      conv(m.trans[b].cout, m.trans[b].C, 1);
    } else {
      const int64_t C = mb.C;
      bn(C);
      const double w_std = std::sqrt(1.0 / static_cast<double>(C));
      for (int64_t i = 0; i < static_cast<int64_t>(desc->classes) * C; ++i)
        *p++ = static_cast<float>(w_std * rng.normal());
      for (int64_t i = 0; i < desc->classes; ++i) *p++ = 0.f;
    }
  }
  if (p - host_params != m.params) return fail(DPB_ACCOUNTING_ERROR, "parameter init count mismatch");
  return DPB_OK;
}

DPB_API void dpb_model_destroy(dpb_model* m) {
  if (!m) return;
  DeviceGuard dg(m->device);
  if (m->graph) cudaGraphExecDestroy(m->graph);
  for (cudaEvent_t e : m->ev) cudaEventDestroy(e);
  if (m->side) cudaStreamDestroy(m->side);
  for (cudaEvent_t e : m->ev_tdone) cudaEventDestroy(e);
  for (cudaEvent_t e : m->ev_bucket) cudaEventDestroy(e);
  if (m->ev_cjoin) cudaEventDestroy(m->ev_cjoin);
  if (m->ev_input) cudaEventDestroy(m->ev_input);
  if (m->cstream) cudaStreamDestroy(m->cstream);
  for (auto& b : m->blocks)
    if (b.blk) destroy(b.blk);
  if (m->mem) {
    cudaFree(m->mem);
    for (int t = 0; t < 6; ++t)
      if (m->mem_tags[t]) m->tracker.free(t, m->mem_tags[t]);
  }
  delete m;
}

DPB_API int dpb_model_create(const dpb_model_desc* desc, int device, void* stream, dpb_model** out) {
  if (out == nullptr) return fail(DPB_CONFIG_ERROR, "null output handle");
  dpb_model* m = new (std::nothrow) dpb_model();
  if (!m) return fail(DPB_CAPACITY_ERROR, "host allocation failed");
  int rc = model_geometry(desc, m);
  if (rc) {
    delete m;
    return rc;
  }
  m->d = *desc;
  m->device = device;
  m->stream = static_cast<cudaStream_t>(stream);
  DeviceGuard dg(device);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete m;
    return cuda_fail(e, "cudaSetDevice");
  }
  const int bk = 4 * desc->k;
  for (auto& b : m->blocks) {
    dpb_block_desc bd{desc->batch, b.h, b.w, b.c0, b.m, desc->k, bk, desc->dtype, DPB_NHWC};
    rc = create(&bd, device, stream, &b.blk, &m->tracker);
    if (rc) {
      dpb_model_destroy(m);
      return rc;
    }
  }
  // device buffers: block inputs and accumulators, transition P / gP, head,
  // split-K partials, BN-backward partials and coefficients
  int64_t bytes = 0;
  int64_t tags[6] = {};
  auto take = [&](int64_t n, int tag = DPB_ARENA_SCRATCH) {  // n floats, accounted under `tag`
    const int64_t o = bytes;
    bytes += (n * 4 + 255) / 256 * 256;
    tags[tag] += bytes - o;
    return o;
  };
  std::vector<int64_t> off;
  for (auto& b : m->blocks) {
    off.push_back(take(b.M * b.Cp, DPB_ARENA_SHARED_GRAD));  // block-output gradient accumulator
  }
  for (auto& t : m->trans) {
    off.push_back(take(t.Mq * t.C, DPB_ARENA_FEATURE_OWNED));  // pooled activations (saved for dW)
    off.push_back(take(t.Mq * t.C, DPB_ARENA_SHARED_GRAD));    // their gradient
    int64_t tchunk;
    off.push_back(take(static_cast<int64_t>(trans_dw_splits(t, tchunk)) * t.cout * t.C));
  }
  const int Cl = m->blocks.back().C;
  const int64_t N = desc->batch;
  const int64_t o_gap = take(N * Cl, DPB_ARENA_FEATURE_OWNED), o_log = take(N * desc->classes, DPB_ARENA_FEATURE_OWNED),
                o_glog = take(N * desc->classes), o_ggap = take(N * Cl, DPB_ARENA_SHARED_GRAD), o_loss = take(N);
  int64_t wmax = static_cast<int64_t>(desc->c0) * desc->in_c * 9, cmax = Cl;
  for (auto& t : m->trans) {
    wmax = std::max<int64_t>(wmax, static_cast<int64_t>(t.cout) * t.C);
    cmax = std::max<int64_t>(cmax, t.C);
  }
  const int64_t stem_splits = (m->blocks[0].M + stem_chunk(desc->c0, desc->in_c) - 1) /
                              stem_chunk(desc->c0, desc->in_c);
  (void)wmax;  // the transitions' dW partials are their own (t.wpart); m->wpart: the stem's
  m->wpart_elems = stem_splits * desc->c0 * desc->in_c * 9;
  if (desc->stem == 1)
    m->wpart_elems = std::max<int64_t>(m->wpart_elems, kStem7Splits * desc->c0 * desc->in_c * kS7Taps);
  int64_t o_y1 = 0, o_arg = 0, o_spart = 0, o_sstat = 0, o_gm = -1, o_s2d = -1, o_ws2d = -1;
  if (desc->stem == 1) {
    m->s2d = StemS2d{desc->in_c, desc->in_h, desc->in_w, m->H1, m->W1};
    const int64_t s2d_rows = desc->batch * m->s2d.rows() * m->s2d.cols() * 2;  // 16-byte rows per plane
    if (desc->dtype == DPB_BF16 && desc->c0 % 8 == 0 && desc->c0 <= tc::kBM && desc->in_c <= 4 &&
        m->blocks[0].Cp % 4 == 0 && s2d_rows < (int64_t{1} << 31)) {
      // the tensor-core stem: space-to-depth planes, forward weights, masked pool gradient
      m->tc_stem = true;
      o_s2d = take(3 * 4 * s2d_rows);
      o_ws2d = take(tc::kBM * 256);  // two fp16 planes of [BN][256]
      o_gm = take(m->M1 * desc->c0);
    }
    o_y1 = take(m->M1 * desc->c0, DPB_ARENA_FEATURE_OWNED);  // stem conv output (reused for its gradient)
    o_arg = take((m->blocks[0].M * desc->c0 + 3) / 4, DPB_ARENA_FEATURE_OWNED);  // max-pool taps
    o_spart = take(4 * m->P1 * desc->c0);
    o_sstat = take(2 * desc->c0);
  }
  const int64_t o_wpart = take(m->wpart_elems);
  m->part_rows = kRowSplitsMax;
  const int64_t o_part = take(4 * kRowSplitsMax * cmax);  // double2 = 4 floats
  const int64_t o_coef = take(2 * cmax);
  const int64_t o_bad = take(1);
  e = cudaMalloc(&m->mem, static_cast<size_t>(bytes));
  if (e != cudaSuccess) {
    dpb_model_destroy(m);
    return cuda_fail(e, "model cudaMalloc");
  }
  for (int t = 0; t < 6; ++t) {
    m->mem_tags[t] = tags[t];
    if (tags[t]) m->tracker.alloc(t, tags[t]);
  }
  char* base = static_cast<char*>(m->mem);
  size_t k = 0;
  for (auto& b : m->blocks) {
    // the block input is written straight into channels [0, c0) of the
    // block's feature arena (row pitch Cp): the block's own pack is skipped
    b.x = static_cast<float*>(b.blk->feat);
    b.acc = reinterpret_cast<float*>(base + off[k++]);
  }
  for (auto& t : m->trans) {
    t.P = reinterpret_cast<float*>(base + off[k++]);
    t.gP = reinterpret_cast<float*>(base + off[k++]);
    t.wpart = reinterpret_cast<float*>(base + off[k++]);
  }
  m->gap = reinterpret_cast<float*>(base + o_gap);
  m->logits = reinterpret_cast<float*>(base + o_log);
  m->g_logits = reinterpret_cast<float*>(base + o_glog);
  m->g_gap = reinterpret_cast<float*>(base + o_ggap);
  m->loss_n = reinterpret_cast<float*>(base + o_loss);
  m->wpart = reinterpret_cast<float*>(base + o_wpart);
  m->part = reinterpret_cast<double2*>(base + o_part);
  m->coef = reinterpret_cast<float*>(base + o_coef);
  m->bad_label = reinterpret_cast<int*>(base + o_bad);
  if (desc->stem == 1) {
    m->y1 = reinterpret_cast<float*>(base + o_y1);
    m->arg = reinterpret_cast<uint8_t*>(base + o_arg);
    m->spart = reinterpret_cast<double2*>(base + o_spart);
    m->sstat = reinterpret_cast<float*>(base + o_sstat);
    if (m->tc_stem) {
      m->gm = reinterpret_cast<float*>(base + o_gm);
      const int64_t rows = desc->batch * m->s2d.rows() * m->s2d.cols() * 2;
      m->xh = reinterpret_cast<uint4*>(base + o_s2d);
      m->xl = m->xh + rows;
      m->xb = m->xl + rows;
      m->wh = reinterpret_cast<__half*>(base + o_ws2d);
      m->wl = m->wh + tc::kBM * 256;
    }
  }
  if (cudaStreamCreateWithFlags(&m->side, cudaStreamNonBlocking) != cudaSuccess) m->side = nullptr;
  cudaEventCreateWithFlags(&m->ev_input, cudaEventDisableTiming);
  for (size_t i = 0; m->side && i < m->trans.size() + 1; ++i) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    m->ev.push_back(e);
  }
  *out = m;
  return DPB_OK;
}

// Gradient buckets in issue order: block b's parameters together with its
// transition's (the head's for the last block) as soon as block b's backward
// is done, last block first; the stem joins block 0.  Registration order makes
// every bucket one contiguous range: [poff(b), poff(b+1)).
static void bucket_ranges(const dpb_model& m, std::vector<std::pair<int64_t, int64_t>>& out) {
  out.clear();
  const int nb = static_cast<int>(m.blocks.size());
  for (int b = nb - 1; b >= 0; --b) {
    const int64_t begin = b == 0 ? 0 : m.blocks[b].poff;
    const int64_t end = b + 1 < nb ? m.blocks[b + 1].poff : m.params;
    out.emplace_back(begin, end);
  }
}

DPB_API int dpb_model_buckets(const dpb_model_desc* desc, int64_t* ranges, int max, int* count) {
  if (!ranges || !count) return fail(DPB_CONFIG_ERROR, "null argument");
  dpb_model m;
  const int rc = model_geometry(desc, &m);
  if (rc) return rc;
  std::vector<std::pair<int64_t, int64_t>> r;
  bucket_ranges(m, r);
  *count = static_cast<int>(r.size());
  for (int i = 0; i < static_cast<int>(r.size()) && i < max; ++i) {
    ranges[2 * i] = r[i].first;
    ranges[2 * i + 1] = r[i].second;
  }
  return DPB_OK;
}

DPB_API int dpb_model_set_comm(dpb_model* m, dpb_comm* comm) {
  if (!m) return fail(DPB_CONFIG_ERROR, "null model");
  DeviceGuard dg(m->device);
  m->comm = reinterpret_cast<dpb::Comm*>(comm);
  if (m->comm && !m->cstream) {
    if (cudaStreamCreateWithFlags(&m->cstream, cudaStreamNonBlocking) != cudaSuccess)
      return fail(DPB_CUDA_ERROR, "communication stream");
    const size_t nb = m->blocks.size();
    m->ev_tdone.resize(m->trans.size());
    m->ev_bucket.resize(nb);
    for (auto& e : m->ev_tdone) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (auto& e : m->ev_bucket) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&m->ev_cjoin, cudaEventDisableTiming);
  }
  if (m->graph) {  // the captured step changes: capture again on the next call
    cudaGraphExecDestroy(m->graph);
    m->graph = nullptr;
  }
  return DPB_OK;
}

DPB_API int dpb_model_wait_input(dpb_model* m, void* stream) {
  if (!m) return fail(DPB_CONFIG_ERROR, "null model");
  DeviceGuard dg(m->device);
  const cudaError_t e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), m->ev_input, 0);
  return e == cudaSuccess ? DPB_OK : cuda_fail(e, "model wait input");
}

DPB_API int dpb_model_memory_stats(dpb_model* m, dpb_memory_stats* out) {
  if (!m || !out) return fail(DPB_CONFIG_ERROR, "null argument");
  m->tracker.snapshot(out);
  return DPB_OK;
}

DPB_API int64_t dpb_model_launch_count(dpb_model* m) {
  if (!m) return -1;
  return m->graph ? m->graph_kernels : m->eager_launches;
}

DPB_API int dpb_model_sync(dpb_model* m) {
  if (!m) return fail(DPB_CONFIG_ERROR, "null model");
  DeviceGuard dg(m->device);
  const cudaError_t e = cudaStreamSynchronize(m->stream);
  if (e != cudaSuccess) return cuda_fail(e, "model sync");
  int bad = 0;
  cudaMemcpy(&bad, m->bad_label, sizeof(int), cudaMemcpyDeviceToHost);
  if (bad) {
    cudaMemset(m->bad_label, 0, sizeof(int));
    return fail(DPB_LABEL_ERROR, "label out of range [0, classes)");
  }
  return DPB_OK;
}

}  // extern "C"

namespace {

// Every launch of one training step on m->stream (and the side stream).
// dpb_model_wait_input's event: an external event node when the step is being
// captured into its graph (so replays record it), a plain record otherwise
static void record_input_event(dpb_model* m, cudaStream_t st) {
  if (!m->ev_input) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(m->ev_input, st, cudaEventRecordExternal);
  else
    cudaEventRecord(m->ev_input, st);
}

int model_step_launch(dpb_model* m, const float* input, const int32_t* labels, const float* params,
                      float* running, float* grads, float* loss) {
  const dpb_model_desc& d = m->d;
  cudaStream_t st = m->stream;
  const int64_t N = d.batch;
  const int nb = static_cast<int>(m->blocks.size());
  // split-K of a reduction over `rows` pixels into at most `smax` chunks of at
  // least `min_chunk` rows (short per-thread chains, many CTAs)
  auto splits_of = [](int64_t rows, int64_t& chunk, int64_t smax = kSplitsMax, int64_t min_chunk = 64) {
    chunk = std::max<int64_t>(min_chunk, (rows + smax - 1) / smax);
    return static_cast<int>((rows + chunk - 1) / chunk);
  };

  // ---- forward --------------------------------------------------------------------
  ModelBlock& b0 = m->blocks[0];
  if (d.stem == 1) {
    const int c0p = (d.c0 + 31) / 32 * 32;
    auto tc_stem = [&](auto tag) {
      using Op = decltype(tag);
      const int64_t pos = N * m->s2d.rows() * m->s2d.cols();
      const int img_blocks = static_cast<int>((pos + 255) / 256);
      launch(k_stem_s2d, img_blocks + Op::BN, 256, 0, st, input, N, m->s2d, params, d.c0, Op::BN, img_blocks,
             m->xh, m->xl, m->xb, m->wh, m->wl);
      const Op op{m->xh, m->xl, reinterpret_cast<const uint4*>(m->wh), reinterpret_cast<const uint4*>(m->wl),
                  m->y1, m->spart, m->s2d, static_cast<int>(d.c0), m->M1};
      launch(tc::tc_gemm_kernel<Op>, dim3(static_cast<unsigned>(m->P1)), tc::kThreads,
             tc::stage_bytes<Op>() + sizeof(int) * tc::kBM, st, op);
    };
    if (m->tc_stem && d.c0 <= 64) {
      tc_stem(StemConvGemm<64>{});  // y and its BN partials in one pass
    } else if (m->tc_stem) {
      tc_stem(StemConvGemm<128>{});
    } else {
      launch(k_stem7_conv, dim3(blocks_of(N * m->H1 * ((m->W1 + 1) / 2), 128), static_cast<unsigned>(c0p / 32)),
             128, sizeof(float) * d.in_c * kS7Taps * c0p, st, input, N, d.in_c, d.in_h, d.in_w, m->H1, m->W1,
             params, d.c0, m->y1);
      launch_channel_partials(st, m->y1, d.c0, m->M1, d.c0, m->spart);
    }
    launch_finalize_stats(st, m->spart, static_cast<int>(m->P1), d.c0, static_cast<double>(m->M1), m->sstat,
                          m->sstat + d.c0);
    launch(k_running, blocks_of(d.c0, 256), 256, 0, st, d.c0, static_cast<const float*>(m->sstat),
           static_cast<const float*>(m->sstat + d.c0), running, running + d.c0);
    if (d.c0 % 4 == 0 && b0.Cp % 4 == 0) {
      launch(k_stem_pool4, blocks_of(b0.M * (d.c0 / 4), 256), 256, 0, st, static_cast<const float*>(m->y1),
             static_cast<int>(b0.M), m->H1, m->W1, b0.h, b0.w, d.c0, static_cast<const float*>(m->sstat),
             static_cast<const float*>(m->sstat + d.c0), params + m->stem_gamma, params + m->stem_beta, b0.x, b0.Cp,
             m->arg);
    } else {
      launch(k_stem_pool, blocks_of(b0.M * d.c0, 256), 256, 0, st, static_cast<const float*>(m->y1), N, m->H1,
             m->W1, b0.h, b0.w, d.c0, static_cast<const float*>(m->sstat),
             static_cast<const float*>(m->sstat + d.c0), params + m->stem_gamma, params + m->stem_beta, b0.x, b0.Cp,
             m->arg);
    }
  } else {
    launch(k_stem_fwd, blocks_of(b0.M, 256), 256, sizeof(float) * d.c0 * d.in_c * 9, st, input, N, d.in_c,
           d.in_h, d.in_w, params, d.c0, b0.x, b0.Cp);
  }
  for (int b = 0; b < nb; ++b) {
    ModelBlock& mb = m->blocks[b];
    int rc = block_forward(mb.blk, mb.x, params + mb.poff, running + mb.roff, 1, 0);
    if (rc) return rc;
    const float* feat = static_cast<const float*>(mb.blk->feat);
    const float* mean = mb.blk->fstat;
    const float* var = mb.blk->fstat + mb.blk->g.Cp;
    if (b + 1 < nb) {
      ModelTrans& t = m->trans[b];
      ModelBlock& nx = m->blocks[b + 1];
      if (t.C % 4 == 0 && mb.Cp % 4 == 0)
        launch(k_trans_pool4, blocks_of(t.Mq * (t.C / 4), 256), 256, 0, st, feat, mb.Cp, t.Mq, mb.h, mb.w, t.C, mean,
               var, params + t.gamma, params + t.beta, t.P);
      else
        launch(k_trans_pool, dim3(blocks_of(t.C, 128), static_cast<unsigned>(std::min<int64_t>(t.Mq, 65535))), 128,
               0, st, feat, mb.Cp, N, mb.h, mb.w, t.C, mean, var, params + t.gamma, params + t.beta, t.P);
      if (d.dtype == DPB_BF16)
        trans_gemm<0>(st, static_cast<int>(t.Mq), t.cout, t.C, t.P, t.C, params + t.w, t.C, nx.x, nx.Cp);
      else
        launch(k_gemm<false, true>, dim3(blocks_of(t.Mq, 64), blocks_of(t.cout, 64), 1), 256, 0, st,
               static_cast<int>(t.Mq), t.cout, t.C, static_cast<const float*>(t.P), t.C, params + t.w, t.C, nx.x,
               nx.Cp, t.C);
      launch(k_running, blocks_of(t.C, 256), 256, 0, st, t.C, mean, var, running + t.run,
             running + t.run + t.C);
    } else {
      const int HW = mb.h * mb.w;
      launch(k_head_gap, blocks_of(N * mb.C, 256), 256, 0, st, feat, mb.Cp, N, HW, mb.C, mean, var,
             params + m->head_gamma, params + m->head_beta, m->gap);
      launch(k_head_logits, blocks_of(((N + kLogitRows - 1) / kLogitRows) * d.classes * 32, 256), 256, 0, st,
             static_cast<const float*>(m->gap), N, mb.C, params + m->head_w, params + m->head_b, d.classes,
             m->logits);
      launch(k_head_loss, static_cast<unsigned>(N), 256, 0, st, static_cast<const float*>(m->gap), N, mb.C,
             params + m->head_w, params + m->head_b, d.classes, labels, m->logits, m->g_logits, m->loss_n,
             m->bad_label);
      launch(k_loss_mean, 1, 32, 0, st, static_cast<const float*>(m->loss_n), N, loss);
      // labels are read; the images too when the stem keeps its own copy (the
      // tensor-core stem's space-to-depth planes) — else after the backward
      if (m->tc_stem) record_input_event(m, st);
      launch(k_running, blocks_of(mb.C, 256), 256, 0, st, mb.C, mean, var, running + m->head_run,
             running + m->head_run + mb.C);
    }
  }

  // ---- backward -------------------------------------------------------------------
  {
    ModelBlock& mb = m->blocks[nb - 1];
    const int C = mb.C, HW = mb.h * mb.w;
    launch(k_head_linear_bwd, blocks_of(N * C + static_cast<int64_t>(d.classes) * C + d.classes, 256), 256, 0,
           st, static_cast<const float*>(m->g_logits), static_cast<const float*>(m->gap), params + m->head_w,
           N, C, d.classes, m->g_gap, grads + m->head_w, grads + m->head_b);
    const float* feat = static_cast<const float*>(mb.blk->feat);
    const float* mean = mb.blk->fstat;
    const float* var = mb.blk->fstat + mb.blk->g.Cp;
    HeadGrad up{m->g_gap, HW, C};
    int64_t chunk;
    const int S = splits_of(mb.M, chunk, kRowSplitsMax, 16);
    launch(k_bnb_partials<HeadGrad>, dim3(S, blocks_of(C, 256)), 256, 0, st, feat, mb.Cp, mb.M, C, mean, var,
           params + m->head_gamma, params + m->head_beta, up, chunk, m->part);
    launch_finalize_bn_bwd(st, m->part, S, C, static_cast<double>(mb.M), grads + m->head_gamma,
                           grads + m->head_beta, m->coef);
    launch(k_bnb_apply<HeadGrad>, dim3(blocks_of(C, 128), static_cast<unsigned>(std::min<int64_t>(mb.M, 65535))),
           128, 0, st, feat, mb.Cp, mb.M, C, mean, var,
           params + m->head_gamma, params + m->head_beta, up, static_cast<const float*>(m->coef), mb.acc, mb.Cp);
  }
  // DP: bucket b = [poff(b), poff(b+1)) (the stem joins block 0), reduced on
  // the communication stream once its gradients exist (dpb_model_buckets)
  const bool dp = m->comm != nullptr;
  auto issue_bucket = [&](int b) -> int {
    const int64_t begin = b == 0 ? 0 : m->blocks[b].poff;
    const int64_t end = b + 1 < nb ? m->blocks[b + 1].poff : m->params;
    cudaEventRecord(m->ev_bucket[b], st);
    cudaStreamWaitEvent(m->cstream, m->ev_bucket[b], 0);
    if (b + 1 < nb && m->side) cudaStreamWaitEvent(m->cstream, m->ev_tdone[b], 0);  // transition b's dW
    return comm_allreduce_avg(m->comm, grads + begin, end - begin, m->cstream);
  };
  for (int b = nb - 1; b >= 0; --b) {
    ModelBlock& mb = m->blocks[b];
    int rc = block_backward(mb.blk, params + mb.poff, mb.acc, grads + mb.poff, mb.Cp);
    if (rc) return rc;
    if (dp && b > 0) {
      rc = issue_bucket(b);
      if (rc) return rc;
    }
    if (b > 0) {
      ModelTrans& t = m->trans[b - 1];
      ModelBlock& pv = m->blocks[b - 1];
      // g_pool = mb.acc[:, :t.cout] (pitch mb.C); dW = g_pool^T . P (split-K), g_P = g_pool . W
      int64_t chunk;
      const int S = trans_dw_splits(t, chunk);
      // dW (gradient-only) on the side stream, overlapping g_P / BN backward and the
      // next block's backward; t.wpart is private to this transition
      cudaStream_t ws = st;
      if (m->side) {
        cudaEventRecord(m->ev[b - 1], st);
        cudaStreamWaitEvent(m->side, m->ev[b - 1], 0);
        ws = m->side;
      }
      if (d.dtype == DPB_BF16) {
        const TransWgradGemm op{mb.acc, t.P, t.wpart, t.cout, t.C, mb.Cp, t.Mq, chunk};
        launch(tc::tc_gemm_kernel<TransWgradGemm>,
               dim3(blocks_of(t.cout, tc::kBM), blocks_of(t.C, TransWgradGemm::BN), S), tc::kThreads,
               tc::stage_bytes<TransWgradGemm>(), ws, op);
      } else {
        launch(k_gemm<true, false>, dim3(blocks_of(t.cout, 64), blocks_of(t.C, 64), S), 256, 0, ws, t.cout, t.C,
               static_cast<int>(t.Mq), static_cast<const float*>(mb.acc), mb.Cp, static_cast<const float*>(t.P),
               t.C, t.wpart, t.C, static_cast<int>(chunk));
      }
      launch_fold_splits(ws, t.wpart, S, static_cast<int64_t>(t.cout) * t.C, grads + t.w);
      if (dp && m->side) cudaEventRecord(m->ev_tdone[b - 1], m->side);
      if (d.dtype == DPB_BF16)
        trans_gemm<1>(st, static_cast<int>(t.Mq), t.C, t.cout, mb.acc, mb.Cp, params + t.w, t.C, t.gP, t.C);
      else
        launch(k_gemm<false, false>, dim3(blocks_of(t.Mq, 64), blocks_of(t.C, 64), 1), 256, 0, st,
               static_cast<int>(t.Mq), t.C, t.cout, static_cast<const float*>(mb.acc), mb.Cp, params + t.w, t.C,
               t.gP, t.C, t.cout);
      const float* feat = static_cast<const float*>(pv.blk->feat);
      const float* mean = pv.blk->fstat;
      const float* var = pv.blk->fstat + pv.blk->g.Cp;
      if (pv.h % 2 == 0 && pv.w % 2 == 0) {  // every pixel in one pooling window: walk the windows
        const int S2 = splits_of(t.Mq, chunk, kRowSplitsMax, 8);
        launch(k_pool_bnb_partials, dim3(S2, blocks_of(t.C, 128)), 128, 0, st, feat, pv.Cp, pv.h, pv.w, t.C,
               mean, var, params + t.gamma, params + t.beta, static_cast<const float*>(t.gP), t.Mq, chunk,
               m->part);
        launch_finalize_bn_bwd(st, m->part, S2, t.C, static_cast<double>(pv.M), grads + t.gamma,
                               grads + t.beta, m->coef);
        launch(k_pool_bnb_apply, dim3(S2, blocks_of(t.C, 128)), 128, 0, st, feat, pv.Cp, pv.h, pv.w, t.C, mean,
               var, params + t.gamma, params + t.beta, static_cast<const float*>(t.gP), t.Mq, chunk,
               static_cast<const float*>(m->coef), pv.acc, pv.Cp);
      } else {
        PoolGrad up{t.gP, pv.h, pv.w, t.C};
        const int S2 = splits_of(pv.M, chunk, kRowSplitsMax, 16);
        launch(k_bnb_partials<PoolGrad>, dim3(S2, blocks_of(t.C, 256)), 256, 0, st, feat, pv.Cp, pv.M, t.C, mean,
               var, params + t.gamma, params + t.beta, up, chunk, m->part);
        launch_finalize_bn_bwd(st, m->part, S2, t.C, static_cast<double>(pv.M), grads + t.gamma,
                               grads + t.beta, m->coef);
        launch(k_bnb_apply<PoolGrad>,
               dim3(blocks_of(t.C, 128), static_cast<unsigned>(std::min<int64_t>(pv.M, 65535))), 128, 0, st, feat,
               pv.Cp, pv.M, t.C, mean, var,
               params + t.gamma, params + t.beta, up, static_cast<const float*>(m->coef), pv.acc, pv.Cp);
      }
    } else if (d.stem == 1) {
      // block-input gradient mb.acc[:, :c0] -> max-pool backward -> ReLU mask
      // -> stem BN backward -> 7x7/2 conv dW (no data gradient, graph.hpp:1170-1181)
      const float* mean = m->sstat;
      const float* var = m->sstat + d.c0;
      int64_t chunk;
      const int S = splits_of(m->M1, chunk, kRowSplitsMax, 16);
      if (m->tc_stem) {
        const int PL = kGatherThreads / (d.c0 / 4);
        launch(k_stem_bnb_gather, S, kGatherThreads, sizeof(double) * 2 * PL * d.c0, st,
               static_cast<const float*>(m->y1), m->M1, m->H1, m->W1, mb.h, mb.w, d.c0, mean, var,
               params + m->stem_gamma, params + m->stem_beta, static_cast<const float*>(mb.acc), mb.Cp,
               static_cast<const uint8_t*>(m->arg), chunk, m->gm, m->part);
      } else {
        launch(k_stem_bnb_partials, dim3(S, blocks_of(d.c0, 32)), 256, 0, st, static_cast<const float*>(m->y1),
               m->M1, m->H1, m->W1, mb.h, mb.w, d.c0, mean, var, params + m->stem_gamma, params + m->stem_beta,
               static_cast<const float*>(mb.acc), mb.Cp, static_cast<const uint8_t*>(m->arg), chunk, m->part);
      }
      launch_finalize_bn_bwd(st, m->part, S, d.c0, static_cast<double>(m->M1), grads + m->stem_gamma,
                             grads + m->stem_beta, m->coef);
      const int64_t pkb = (m->M1 + tc::kBK - 1) / tc::kBK;
      if (m->tc_stem) {
        const int64_t per = (pkb + kStem7Splits - 1) / kStem7Splits;
        const int S7 = static_cast<int>((pkb + per - 1) / per);
        const StemWgradGemm op{m->xb, m->y1, m->gm, mean, var, params + m->stem_gamma, params + m->stem_beta,
                               m->coef, m->wpart, m->s2d, static_cast<int>(d.c0), m->M1, per * tc::kBK};
        launch(tc::tc_gemm_kernel<StemWgradGemm>, dim3(1, 1, static_cast<unsigned>(S7)), tc::kThreads,
               tc::stage_bytes<StemWgradGemm>() + sizeof(float) * 6 * tc::kBM + sizeof(int) * tc::kBK, st, op);
        launch_fold_splits(st, m->wpart, S7, static_cast<int64_t>(d.c0) * d.in_c * kS7Taps, grads);
      } else {
      const int ty7 = (m->H1 + kS7TH - 1) / kS7TH, tx7 = (m->W1 + kS7TW - 1) / kS7TW;
      const int64_t ntiles = N * ty7 * tx7;
      const int64_t per = (ntiles + kStem7Splits - 1) / kStem7Splits;
      const int S7 = static_cast<int>((ntiles + per - 1) / per);
      const int th = (stem7_tiles(d.c0, d.in_c) + 31) / 32 * 32;
      launch(k_stem7_wgrad, S7, th, sizeof(float) * stem7_wgrad_smem_floats(d.c0, d.in_c), st, input, N, d.in_c,
             d.in_h, d.in_w, m->H1, m->W1, static_cast<const float*>(m->y1), d.c0, mean, var,
             params + m->stem_gamma, params + m->stem_beta, static_cast<const float*>(mb.acc), mb.Cp, mb.h, mb.w,
             static_cast<const uint8_t*>(m->arg), static_cast<const float*>(m->coef), per, m->wpart);
      launch_fold_splits(st, m->wpart, S7, static_cast<int64_t>(d.c0) * d.in_c * kS7Taps, grads);
      }
    } else {
      const int chunk = stem_chunk(d.c0, d.in_c);
      const int S = static_cast<int>((mb.M + chunk - 1) / chunk);
      launch(k_stem_wgrad, S, 256, sizeof(float) * chunk * (d.c0 + d.in_c * 9), st, input, N, d.in_c,
             d.in_h, d.in_w, static_cast<const float*>(mb.acc), mb.Cp, d.c0, m->wpart);
      launch_fold_splits(st, m->wpart, S, static_cast<int64_t>(d.c0) * d.in_c * 9, grads);
    }
    if (dp && b == 0) {
      rc = issue_bucket(0);
      if (rc) return rc;
    }
  }
  if (m->side && !m->trans.empty()) {  // join: the caller's stream sees every gradient
    cudaEventRecord(m->ev.back(), m->side);
    cudaStreamWaitEvent(st, m->ev.back(), 0);
  }
  if (dp) {  // ... averaged over the ranks
    cudaEventRecord(m->ev_cjoin, m->cstream);
    cudaStreamWaitEvent(st, m->ev_cjoin, 0);
  }
  const cudaError_t e = cudaGetLastError();
  if (!m->tc_stem) record_input_event(m, st);
  return e == cudaSuccess ? DPB_OK : cuda_fail(e, "model step launch");
}

}  // namespace

extern "C" {

// The step is ~700 launches; replaying them as one CUDA graph removes the
// per-launch host cost and the gaps it leaves on the device.  The graph is
// captured on the first call and replayed while (input, labels, params,
// running, grads, loss) are the same buffers; the stream must be a created
// stream that is not itself being captured (a caller capturing its own graph,
// or the legacy default stream, gets the eager launches).  DPB_MODEL_NO_GRAPH=1
// always launches eagerly.
DPB_API int dpb_model_step(dpb_model* m, const float* input, const int32_t* labels, const float* params,
                           float* running, float* grads, float* loss) {
  if (!m || !input || !labels || !params || !running || !grads || !loss)
    return fail(DPB_CONFIG_ERROR, "null pointer argument");
  DeviceGuard dg(m->device);
  cudaStream_t st = m->stream;
  static const bool no_graph = std::getenv("DPB_MODEL_NO_GRAPH") != nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const bool legacy = st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread;
  if (no_graph || legacy || cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
  {
    const int64_t c0 = launch_counter();
    const int rc = model_step_launch(m, input, labels, params, running, grads, loss);
    m->eager_launches = launch_counter() - c0;
    return rc;
  }
  const void* key[6] = {input, labels, params, running, grads, loss};
  if (m->graph == nullptr || std::memcmp(key, m->graph_key, sizeof(key)) != 0) {
    if (m->graph) {
      cudaGraphExecDestroy(m->graph);
      m->graph = nullptr;
    }
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "model step capture");
    const int rc = model_step_launch(m, input, labels, params, running, grads, loss);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(st, &g);
    if (rc != DPB_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "model step capture");
    {
      size_t nn = 0;
      cudaGraphGetNodes(g, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(g, nodes.data(), &nn);
      int64_t kern = 0;
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        cudaGraphNodeGetType(nd, &ty);
        kern += ty == cudaGraphNodeTypeKernel;
      }
      m->graph_kernels = kern;
    }
    e = cudaGraphInstantiate(&m->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      m->graph = nullptr;
      return cuda_fail(e, "model step graph instantiate");
    }
    std::memcpy(m->graph_key, key, sizeof(key));
  }
  const cudaError_t e = cudaGraphLaunch(m->graph, st);
  return e == cudaSuccess ? DPB_OK : cuda_fail(e, "model step graph launch");
}

}  // extern "C"
