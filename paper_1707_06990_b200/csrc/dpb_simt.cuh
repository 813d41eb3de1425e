// SIMT implicit-GEMM engine for the dense block (fp32 FMA, fp32 accumulate).
//
// One generic 256-thread tiled kernel; each convolution of the layer is an
// "Op" that supplies
//   * prologue():   per-channel BN coefficients into dynamic shared memory,
//   * load_a/b():   the operand producers — BN+ReLU recompute, 3x3 halo
//                   gather with zero padding AFTER activation, BN-backward
//                   transform — fused so concat / act_a / act_b / t1 are
//                   never materialised in HBM (the paper's shared storage
//                   taken to its limit: Shared1 = Shared2 = 0),
//   * epilogue():   stores plus per-column reductions (BN statistics or BN
//                   backward sums) written as per-CTA fp64 partials that a
//                   fixed-order finalize kernel folds deterministically.
// This is the fp32 parity path (1e-4) and the bf16-storage reference path;
// the tcgen05 kernels (dpb_tc.cuh) replace the bf16 hot GEMMs.
#pragma once

#include "dpb_common.cuh"

namespace dpb {

constexpr int kThreads = 256;
constexpr int kBK = 16;

template <int BM, int BN, class Op>
__global__ void __launch_bounds__(kThreads) gemm_kernel(Op op) {
  constexpr int TM = BM / 16;
  constexpr int TN = BN / 16;
  __shared__ float As[kBK][BM + 4];
  __shared__ float Bs[kBK][BN + 4];
  extern __shared__ float4 dyn4[];
  char* dyn = reinterpret_cast<char*>(dyn4);
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  pdl_enter();
  op.prologue(dyn, n0);
  __syncthreads();
  int64_t kbeg, kend;
  op.k_range(blockIdx.z, kbeg, kend);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = kbeg; k0 < kend; k0 += kBK) {
    for (int e = tid; e < BM * kBK; e += kThreads) {
      int kk, mm;
      if (Op::kAKFast) { kk = e % kBK; mm = e / kBK; }
      else { mm = e % BM; kk = e / BM; }
      const int64_t gk = k0 + kk, gm = m0 + mm;
      As[kk][mm] = (gk < kend && gm < op.rows()) ? op.load_a(dyn, n0, gm, gk) : 0.f;
    }
    for (int e = tid; e < BN * kBK; e += kThreads) {
      int kk, nn;
      if (Op::kBKFast) { kk = e % kBK; nn = e / kBK; }
      else { nn = e % BN; kk = e / BN; }
      const int64_t gk = k0 + kk;
      const int gn = n0 + nn;
      Bs[kk][nn] = (gk < kend && gn < op.cols()) ? op.load_b(dyn, gk, gn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  if constexpr (Op::kColStats) {
    // epilogue with per-column (s1, s2) reduction
    __shared__ double red1[16][BN];
    __shared__ double red2[16][BN];
    double s1[TN], s2[TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) { s1[j] = 0.0; s2[j] = 0.0; }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t gm = m0 + ty * TM + i;
      if (gm >= op.rows()) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int gn = n0 + tx * TN + j;
        if (gn >= op.cols()) continue;
        double a = 0.0, b = 0.0;
        op.epilogue(dyn, n0, gm, gn, acc[i][j], a, b);
        s1[j] += a;
        s2[j] += b;
      }
    }
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      red1[ty][tx * TN + j] = s1[j];
      red2[ty][tx * TN + j] = s2[j];
    }
    __syncthreads();
    if (tid < BN && n0 + tid < op.cols()) {
      double a = 0.0, b = 0.0;
      for (int r = 0; r < 16; ++r) { a += red1[r][tid]; b += red2[r][tid]; }
      double2* part = op.partials() + static_cast<int64_t>(blockIdx.x) * op.cols();
      part[n0 + tid] = make_double2(a, b);
    }
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t gm = m0 + ty * TM + i;
      if (gm >= op.rows()) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int gn = n0 + tx * TN + j;
        if (gn >= op.cols()) continue;
        op.store(gm, gn, acc[i][j]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Layer arguments shared by every op of one bottleneck layer.
template <typename S>
struct LayerArgs {
  int64_t M;      // pixels N*H*W (GEMM rows)
  int H, W;       // spatial extent for 3x3 neighbourhoods
  int C;          // feature-arena row pitch (block output channels, padded to 4)
  int Ca;         // row pitch of the accumulator acc
  int c;          // this layer's input channels (concat prefix)
  int cg;         // row pitch of g1 (c padded to 4)
  int bk, k;      // bottleneck width, growth rate
  S* feat;        // [M, C]  NHWC features
  S* z;           // [M, bk] this layer's bottleneck output
  const float* gamma_a; const float* beta_a; const float* w1;  // flat params
  const float* gamma_b; const float* beta_b; const float* w2;
  const float* amean;   // BN_a statistics of this layer: mean[c], var[c]
  const float* avar;    //   (train: the shared feature-channel stats, F6)
  const float* bmean;   // BN_b statistics: mean[bk], var[bk]
  const float* bvar;
  float* acc;           // [M, C] fp32 block-gradient accumulator
  float* g0;            // [M, bk] fp32 masked 3x3 dgrad (t0)
  float* g1;            // [M, c]  fp32 masked 1x1 dgrad (t2)
  const float* bnb_bwd; // [bk][2] mg, mgx of BN_b backward
  double2* part;        // per-CTA partial sums
  float* wpart;         // split-K weight-gradient partials
  int64_t kchunk;       // pixels per split for the wgrad ops
};

__device__ __forceinline__ void fill_bn_fwd(BnFwd* t, int count, int first,
                                            const float* mean_p, const float* var_p,
                                            const float* gamma, const float* beta) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const int ch = first + i;
    const float mean = mean_p[ch], var = var_p[ch];
    const float inv = bn_inv(var);
    t[i] = BnFwd{mean, gamma[ch] * inv, beta[ch], inv, gamma[ch]};
  }
}

__device__ __forceinline__ void fill_bn_aff(BnAff* t, int count, int first, const float* mean_p,
                                            const float* var_p, const float* gamma,
                                            const float* beta) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const int ch = first + i;
    const float scale = gamma[ch] * bn_inv(var_p[ch]);
    t[i] = BnAff{scale, fmaf(-mean_p[ch], scale, beta[ch])};
  }
}

__device__ __forceinline__ float bn_relu(const BnFwd& b, float x) {
  const float t = fmaf(x - b.mean, b.scale, b.beta);
  return t > 0.f ? t : 0.f;
}

// tap t in [0,9): (dy, dx) = (t/3 - 1, t%3 - 1)
__device__ __forceinline__ bool shifted(int64_t p, int H, int W, int dy, int dx,
                                        int64_t& q) {
  const int x = static_cast<int>(p % W);
  const int y = static_cast<int>((p / W) % H);
  const int yy = y + dy, xx = x + dx;
  if (yy < 0 || yy >= H || xx < 0 || xx >= W) return false;
  q = p + static_cast<int64_t>(dy) * W + dx;
  return true;
}

// ---- forward: z = relu(bn_a(cat)) . W1^T  (+ BN_b statistics partials) ----
template <typename S>
struct Conv1x1Fwd {
  LayerArgs<S> a;
  static constexpr bool kAKFast = true, kBKFast = true, kColStats = true;
  __device__ int64_t rows() const { return a.M; }
  __device__ int cols() const { return a.bk; }
  __device__ void k_range(int, int64_t& b, int64_t& e) const { b = 0; e = a.c; }
  __device__ double2* partials() const { return a.part; }
  static size_t smem(const LayerArgs<S>& a) { return sizeof(BnFwd) * a.c; }
  __device__ void prologue(char* d, int) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(d), a.c, 0, a.amean, a.avar, a.gamma_a, a.beta_a);
  }
  __device__ float load_a(const char* d, int, int64_t m, int64_t kk) const {
    return bn_relu(reinterpret_cast<const BnFwd*>(d)[kk], to_f(a.feat[m * a.C + kk]));
  }
  __device__ float load_b(const char*, int64_t kk, int n) const {
    return a.w1[static_cast<int64_t>(n) * a.c + kk];
  }
  __device__ void epilogue(const char*, int, int64_t m, int n, float v, double& s1,
                           double& s2) const {
    const S r = from_f<S>(v);
    a.z[m * a.bk + n] = r;
    const double f = to_f(r);
    s1 = f;
    s2 = f * f;
  }
  __device__ void store(int64_t, int, float) const {}
};

// ---- forward: y = conv3x3(relu(bn_b(z))) -> feat[:, c:c+k] (+ stats) ------
template <typename S>
struct Conv3x3Fwd {
  LayerArgs<S> a;
  static constexpr bool kAKFast = true, kBKFast = true, kColStats = true;
  __device__ int64_t rows() const { return a.M; }
  __device__ int cols() const { return a.k; }
  __device__ void k_range(int, int64_t& b, int64_t& e) const { b = 0; e = 9 * a.bk; }
  __device__ double2* partials() const { return a.part; }
  static size_t smem(const LayerArgs<S>& a) { return sizeof(BnFwd) * a.bk; }
  __device__ void prologue(char* d, int) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(d), a.bk, 0, a.bmean, a.bvar, a.gamma_b, a.beta_b);
  }
  __device__ float load_a(const char* d, int, int64_t m, int64_t kk) const {
    const int tap = static_cast<int>(kk / a.bk);
    const int j = static_cast<int>(kk - static_cast<int64_t>(tap) * a.bk);
    int64_t q;
    if (!shifted(m, a.H, a.W, tap / 3 - 1, tap % 3 - 1, q)) return 0.f;  // pad after act
    return bn_relu(reinterpret_cast<const BnFwd*>(d)[j], to_f(a.z[q * a.bk + j]));
  }
  __device__ float load_b(const char*, int64_t kk, int o) const {
    const int tap = static_cast<int>(kk / a.bk);
    const int j = static_cast<int>(kk - static_cast<int64_t>(tap) * a.bk);
    return a.w2[(static_cast<int64_t>(o) * a.bk + j) * 9 + tap];
  }
  __device__ void epilogue(const char*, int, int64_t m, int o, float v, double& s1,
                           double& s2) const {
    const S r = from_f<S>(v);
    a.feat[m * a.C + a.c + o] = r;
    const double f = to_f(r);
    s1 = f;
    s2 = f * f;
  }
  __device__ void store(int64_t, int, float) const {}
};

// ---- backward: t0 = relu'(act_b) * dgrad3x3(acc[:, c:c+k])  (+ BN_b sums) --
template <typename S>
struct Conv3x3Dgrad {
  LayerArgs<S> a;
  static constexpr bool kAKFast = true, kBKFast = false, kColStats = true;
  __device__ int64_t rows() const { return a.M; }
  __device__ int cols() const { return a.bk; }
  __device__ void k_range(int, int64_t& b, int64_t& e) const { b = 0; e = 9 * a.k; }
  __device__ double2* partials() const { return a.part; }
  static size_t smem(const LayerArgs<S>& a) { return sizeof(BnFwd) * a.bk; }
  __device__ void prologue(char* d, int) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(d), a.bk, 0, a.bmean, a.bvar, a.gamma_b, a.beta_b);
  }
  __device__ float load_a(const char*, int, int64_t m, int64_t kk) const {
    const int tap = static_cast<int>(kk / a.k);
    const int o = static_cast<int>(kk - static_cast<int64_t>(tap) * a.k);
    int64_t q;  // dx[p] = sum_tap dy[p - d_tap] W[tap]
    if (!shifted(m, a.H, a.W, 1 - tap / 3, 1 - tap % 3, q)) return 0.f;
    return a.acc[q * a.Ca + a.c + o];
  }
  __device__ float load_b(const char*, int64_t kk, int j) const {
    const int tap = static_cast<int>(kk / a.k);
    const int o = static_cast<int>(kk - static_cast<int64_t>(tap) * a.k);
    return a.w2[(static_cast<int64_t>(o) * a.bk + j) * 9 + tap];
  }
  __device__ void epilogue(const char* d, int, int64_t m, int j, float v, double& s1,
                           double& s2) const {
    const BnFwd b = reinterpret_cast<const BnFwd*>(d)[j];
    const float zv = to_f(a.z[m * a.bk + j]);
    const float g = relu_mask_ref(b, zv) ? v : 0.f;  // relu_backward by act_b (ops.hpp:268-287)
    a.g0[m * a.bk + j] = g;
    const float xh = (zv - b.mean) * b.inv;
    s1 = g;
    s2 = static_cast<double>(g) * xh;
  }
  __device__ void store(int64_t, int, float) const {}
};

// ---- backward: dW2 partials = act_b(shifted)^T . dY, split over pixels ----
template <typename S>
struct Conv3x3Wgrad {
  LayerArgs<S> a;
  static constexpr bool kAKFast = false, kBKFast = false, kColStats = false;
  __device__ int64_t rows() const { return 9 * a.bk; }
  __device__ int cols() const { return a.k; }
  __device__ void k_range(int z, int64_t& b, int64_t& e) const {
    b = static_cast<int64_t>(z) * a.kchunk;
    e = b + a.kchunk < a.M ? b + a.kchunk : a.M;
  }
  __device__ double2* partials() const { return nullptr; }
  static size_t smem(const LayerArgs<S>& a) { return sizeof(BnFwd) * a.bk; }
  __device__ void prologue(char* d, int) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(d), a.bk, 0, a.bmean, a.bvar, a.gamma_b, a.beta_b);
  }
  __device__ float load_a(const char* d, int, int64_t r, int64_t p) const {
    const int tap = static_cast<int>(r / a.bk);
    const int j = static_cast<int>(r - static_cast<int64_t>(tap) * a.bk);
    int64_t q;
    if (!shifted(p, a.H, a.W, tap / 3 - 1, tap % 3 - 1, q)) return 0.f;
    return bn_relu(reinterpret_cast<const BnFwd*>(d)[j], to_f(a.z[q * a.bk + j]));
  }
  __device__ float load_b(const char*, int64_t p, int o) const {
    return a.acc[p * a.Ca + a.c + o];
  }
  __device__ void epilogue(const char*, int, int64_t, int, float, double&, double&) const {}
  __device__ void store(int64_t r, int o, float v) const {
    a.wpart[(static_cast<int64_t>(blockIdx.z) * 9 * a.bk + r) * a.k + o] = v;
  }
};

// t1 = BN_b backward of t0 against x = z (ops.hpp:236-242), recomputed
__device__ __forceinline__ float bnb_t1(const BnBwd& b, float g, float x) {
  const float xh = (x - b.mean) * b.inv;
  return b.ginv * (g - b.mg - xh * b.mgx);
}

template <typename S>
__device__ __forceinline__ void fill_bn_bwd(BnBwd* t, const LayerArgs<S>& a) {
  for (int j = threadIdx.x; j < a.bk; j += blockDim.x) {
    const float inv = bn_inv(a.bvar[j]);
    t[j] = BnBwd{a.bmean[j], inv, a.gamma_b[j] * inv, a.bnb_bwd[2 * j],
                 a.bnb_bwd[2 * j + 1]};
  }
}

// ---- backward: t2 = relu'(act_a) * (t1 . W1)  (+ BN_a sums) ----------------
template <typename S, int BN>
struct Conv1x1Dgrad {
  LayerArgs<S> a;
  static constexpr bool kAKFast = true, kBKFast = false, kColStats = true;
  __device__ int64_t rows() const { return a.M; }
  __device__ int cols() const { return a.c; }
  __device__ void k_range(int, int64_t& b, int64_t& e) const { b = 0; e = a.bk; }
  __device__ double2* partials() const { return a.part; }
  static size_t smem(const LayerArgs<S>& a) {
    return sizeof(BnBwd) * a.bk + sizeof(BnFwd) * BN + 16;
  }
  __device__ const BnFwd* tile_a(const char* d) const {
    return reinterpret_cast<const BnFwd*>(d + ((sizeof(BnBwd) * a.bk + 15) / 16) * 16);
  }
  __device__ void prologue(char* d, int n0) const {
    fill_bn_bwd(reinterpret_cast<BnBwd*>(d), a);
    BnFwd* t = const_cast<BnFwd*>(tile_a(d));
    const int cnt = a.c - n0 < BN ? a.c - n0 : BN;
    fill_bn_fwd(t, cnt, n0, a.amean, a.avar, a.gamma_a, a.beta_a);
  }
  __device__ float load_a(const char* d, int, int64_t m, int64_t j) const {
    return bnb_t1(reinterpret_cast<const BnBwd*>(d)[j], a.g0[m * a.bk + j],
                  to_f(a.z[m * a.bk + j]));
  }
  __device__ float load_b(const char*, int64_t j, int i) const {
    return a.w1[j * a.c + i];
  }
  __device__ void epilogue(const char* d, int n0, int64_t m, int i, float v,
                           double& s1, double& s2) const {
    const BnFwd b = tile_a(d)[i - n0];
    const float x = to_f(a.feat[m * a.C + i]);
    const float g = relu_mask_ref(b, x) ? v : 0.f;
    a.g1[m * a.cg + i] = g;
    const float xh = (x - b.mean) * b.inv;
    s1 = g;
    s2 = static_cast<double>(g) * xh;
  }
  __device__ void store(int64_t, int, float) const {}
};

// ---- backward: dW1 partials = t1^T . act_a, split over pixels -------------
template <typename S, int BN>
struct Conv1x1Wgrad {
  LayerArgs<S> a;
  static constexpr bool kAKFast = false, kBKFast = false, kColStats = false;
  __device__ int64_t rows() const { return a.bk; }
  __device__ int cols() const { return a.c; }
  __device__ void k_range(int z, int64_t& b, int64_t& e) const {
    b = static_cast<int64_t>(z) * a.kchunk;
    e = b + a.kchunk < a.M ? b + a.kchunk : a.M;
  }
  __device__ double2* partials() const { return nullptr; }
  static size_t smem(const LayerArgs<S>& a) {
    return sizeof(BnBwd) * a.bk + sizeof(BnFwd) * BN + 16;
  }
  __device__ const BnFwd* tile_a(const char* d) const {
    return reinterpret_cast<const BnFwd*>(d + ((sizeof(BnBwd) * a.bk + 15) / 16) * 16);
  }
  __device__ void prologue(char* d, int n0) const {
    fill_bn_bwd(reinterpret_cast<BnBwd*>(d), a);
    BnFwd* t = const_cast<BnFwd*>(tile_a(d));
    const int cnt = a.c - n0 < BN ? a.c - n0 : BN;
    fill_bn_fwd(t, cnt, n0, a.amean, a.avar, a.gamma_a, a.beta_a);
  }
  __device__ float load_a(const char* d, int, int64_t j, int64_t p) const {
    return bnb_t1(reinterpret_cast<const BnBwd*>(d)[j], a.g0[p * a.bk + j],
                  to_f(a.z[p * a.bk + j]));
  }
  __device__ float load_b(const char* d, int64_t p, int i) const {
    return bn_relu(tile_a(d)[i - blockIdx.y * BN], to_f(a.feat[p * a.C + i]));
  }
  __device__ void epilogue(const char*, int, int64_t, int, float, double&, double&) const {}
  __device__ void store(int64_t j, int i, float v) const {
    a.wpart[(static_cast<int64_t>(blockIdx.z) * a.bk + j) * a.c + i] = v;
  }
};

}  // namespace dpb
