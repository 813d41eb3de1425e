// The six convolutions of one bottleneck layer as tcgen05 implicit GEMMs.
//
//   op          M (tile 128)   N (BN)      K              operands (A/B major)
//   Tc1x1Fwd    pixels         bk          c    (split)   act_a K / W1 K
//   Tc3x3Fwd    pixels         k (pad 16)  9*bk (split)   act_b(shifted) K / W2 K
//   Tc3x3Dgrad  pixels         bk          9*kp           dY(shifted) K / W2 K
//   Tc1x1Dgrad  pixels         c tile      bk             t1 K / W1 MN
//   Tc1x1Wgrad  channels c     bk          pixels (split) act_a MN / t1 MN
//   Tc3x3Wgrad  (tap, j) 9*bk  k (pad 16)  pixels (split) act_b(shifted) MN / dY MN
//
// Producers recompute BN+ReLU (act_a, act_b) and the BN_b backward (t1) on
// the fly — the paper's recompute-on-backward with no Shared1/Shared2
// buffers — and zero the 3x3 padding AFTER the activation.  Epilogues apply
// the ReLU masks and emit the BN reduction partials.  Reference semantics:
// /root/reference/proj/include/denseplan/graph.hpp:618-670 (forward) and
// :856-945 (backward); ops.hpp:115-134, 206-243, 268-287, 315-387.
#pragma once

#include "dpb_simt.cuh"  // LayerArgs, BnFwd/BnBwd helpers
#include "dpb_tc.cuh"

namespace dpb {
namespace tc {

// Per-launch flags.
struct TcArgs {
  LayerArgs<float> a;
  int kp;           // k rounded up to 8 (per-tap K stride of the 3x3 dgrad)
  int vec;          // feature / accumulator rows are 16-byte aligned at c
  int n0_unused;
};

// (y << 16 | x) of the CTA's 128 pixel rows, computed once in the prologue so
// the 3x3 producers never divide.
__device__ __forceinline__ void fill_row_yx(int* yx, int64_t m0, int64_t M, int H, int W) {
  for (int r = threadIdx.x; r < kBM; r += kThreads) {
    const int64_t p = m0 + r;
    int v = 0;
    if (p < M) {
      const int pix = static_cast<int>(p % (static_cast<int64_t>(H) * W));
      v = ((pix / W) << 16) | (pix % W);
    }
    yx[r] = v;
  }
}

// Neighbour pixel p + (dy, dx) of a row with coordinates yx; false when it
// falls in the zero padding.
__device__ __forceinline__ bool neighbour(int64_t p, int yx, int H, int W, int dy, int dx,
                                          int64_t& q) {
  const int y = (yx >> 16) + dy, x = (yx & 0xFFFF) + dx;
  if (y < 0 || y >= H || x < 0 || x >= W) return false;
  q = p + static_cast<int64_t>(dy) * W + dx;
  return true;
}

__device__ __forceinline__ void bnrelu8(const BnFwd* t, int ch0, int nvalid, float (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = i < nvalid ? bn_relu(t[ch0 + i], v[i]) : 0.f;
}

template <bool SPLIT>
__device__ __forceinline__ void put8(uint8_t* hi, uint8_t* lo, uint32_t off, const float (&v)[8]) {
  if constexpr (SPLIT) {  // forward operands: fp16x3 (split8_h)
    uint4 h, l;
    split8_h(v, h, l);
    st_shared16(hi, off, h);
    st_shared16(lo, off, l);
  } else {
    st_shared16(hi, off, to_bf16x8(v));
  }
}

// ---- forward 1x1: z = relu(bn_a(x)) . W1^T, bf16x3 -------------------------------
template <int BN_>
struct Tc1x1Fwd {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = true, kColSums = true, kF16 = true;
  static constexpr int kAMN = 0, kBMN = 0;
  TcArgs t;
  __device__ int num_kb() const { return (t.a.c + kBK - 1) / kBK; }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_aff(reinterpret_cast<BnAff*>(aux), t.a.c, 0, t.a.amean, t.a.avar, t.a.gamma_a,
                t.a.beta_a);
  }
  __device__ void produce(uint8_t* ah, uint8_t* al, uint8_t* bh, uint8_t* bl, int kb,
                          const uint8_t* aux) const {
    const LayerArgs<float>& a = t.a;
    const BnAff* bn = reinterpret_cast<const BnAff*>(aux);
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;
#pragma unroll
    for (int q = threadIdx.x; q < kBM * kBK / 8; q += kThreads) {
      int row, kc;
      kmajor_coords(q, row, kc);
      const int ch0 = kb * kBK + kc;
      const int64_t p = m0 + row;
      float v[8];
      const int nv = a.c - ch0;
      if (p < a.M && nv > 0) {
        load8(a.feat + p * a.C + ch0, nv, t.vec, v);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = i < nv ? fmaxf(fmaf(v[i], bn[ch0 + i].scale, bn[ch0 + i].shift), 0.f) : 0.f;
      } else {
        zero8(v);
      }
      put8<true>(ah, al, Tile<kBM>::kmajor_chunk(row, kc), v);
    }
#pragma unroll
    for (int q = threadIdx.x; q < BN * kBK / 8; q += kThreads) {
      int row, kc;
      kmajor_coords(q, row, kc);
      const int i0 = kb * kBK + kc;
      float v[8];
      if (row < a.bk && i0 < a.c) load8(a.w1 + static_cast<int64_t>(row) * a.c + i0, a.c - i0, false, v);
      else zero8(v);
      put8<true>(bh, bl, Tile<BN>::kmajor_chunk(row, kc), v);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&s1)[8],
                           float (&s2)[8]) const {
    const LayerArgs<float>& a = t.a;
    const int64_t p = static_cast<int64_t>(blockIdx.x) * kBM + row;
    const int nv = p < a.M ? a.bk - col0 : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = i < nv;
      s1[i] = ok ? v[i] : 0.f;
      s2[i] = ok ? v[i] * v[i] : 0.f;
    }
    if (nv > 0) store8(a.z + p * a.bk + col0, nv, (a.bk & 3) == 0, v);
  }
  __device__ void col_sums(int c, double s1, double s2) const {
    if (c < t.a.bk) t.a.part[static_cast<int64_t>(blockIdx.x) * t.a.bk + c] = make_double2(s1, s2);
  }
};

// ---- forward 3x3: y = conv3x3(relu(bn_b(z))) -> feat[:, c:c+k], bf16x3 -----------
template <int BN_>
struct Tc3x3Fwd {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = true, kColSums = true, kF16 = true;
  static constexpr int kAMN = 0, kBMN = 0;
  TcArgs t;
  __device__ int num_kb() const { return (9 * t.a.bk + kBK - 1) / kBK; }
  __device__ const int* row_yx(const uint8_t* aux) const {
    return reinterpret_cast<const int*>(aux + sizeof(BnFwd) * t.a.bk);
  }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(aux), t.a.bk, 0, t.a.bmean, t.a.bvar, t.a.gamma_b,
                t.a.beta_b);
    fill_row_yx(const_cast<int*>(row_yx(aux)), static_cast<int64_t>(blockIdx.x) * kBM, t.a.M,
                t.a.H, t.a.W);
  }
  __device__ void produce(uint8_t* ah, uint8_t* al, uint8_t* bh, uint8_t* bl, int kb,
                          const uint8_t* aux) const {
    const LayerArgs<float>& a = t.a;
    const BnFwd* bn = reinterpret_cast<const BnFwd*>(aux);
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;
    const int K = 9 * a.bk;
#pragma unroll
    for (int q = threadIdx.x; q < kBM * kBK / 8; q += kThreads) {
      int row, kc;
      kmajor_coords(q, row, kc);
      const int k0 = kb * kBK + kc;
      const int64_t p = m0 + row;
      float v[8];
      zero8(v);
      if (p < a.M && k0 < K) {
        const int tap = k0 / a.bk, j0 = k0 - tap * a.bk;
        int64_t nb;
        // bk % 8 == 0 (checked at dispatch): a chunk never straddles taps
        if (neighbour(p, row_yx(aux)[row], a.H, a.W, tap / 3 - 1, tap % 3 - 1, nb)) {
          load8(a.z + nb * a.bk + j0, 8, (a.bk & 3) == 0, v);
          bnrelu8(bn, j0, 8, v);
        }
      }
      put8<true>(ah, al, Tile<kBM>::kmajor_chunk(row, kc), v);
    }
#pragma unroll
    for (int q = threadIdx.x; q < BN * kBK / 8; q += kThreads) {
      int o, kc;
      kmajor_coords(q, o, kc);
      const int k0 = kb * kBK + kc;
      float v[8];
      zero8(v);
      if (o < a.k && k0 < K) {
        const int tap = k0 / a.bk, j0 = k0 - tap * a.bk;
        const float* w = a.w2 + (static_cast<int64_t>(o) * a.bk + j0) * 9 + tap;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldg(w + 9 * i);
      }
      put8<true>(bh, bl, Tile<BN>::kmajor_chunk(o, kc), v);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&s1)[8],
                           float (&s2)[8]) const {
    const LayerArgs<float>& a = t.a;
    const int64_t p = static_cast<int64_t>(blockIdx.x) * kBM + row;
    const int nv = p < a.M ? a.k - col0 : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = i < nv;
      s1[i] = ok ? v[i] : 0.f;
      s2[i] = ok ? v[i] * v[i] : 0.f;
    }
    if (nv > 0) store8(a.feat + p * a.C + a.c + col0, nv, t.vec, v);
  }
  __device__ void col_sums(int c, double s1, double s2) const {
    if (c < t.a.k) t.a.part[static_cast<int64_t>(blockIdx.x) * t.a.k + c] = make_double2(s1, s2);
  }
};

// ---- backward 3x3 dgrad: t0 = relu'(act_b) * conv3x3^T(dY), bf16 -------------------
template <int BN_>
struct Tc3x3Dgrad {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = false, kColSums = true, kF16 = false;
  static constexpr int kAMN = 0, kBMN = 0;
  TcArgs t;
  __device__ int num_kb() const { return (9 * t.kp + kBK - 1) / kBK; }
  __device__ const int* row_yx(const uint8_t* aux) const {
    return reinterpret_cast<const int*>(aux + sizeof(BnFwd) * t.a.bk);
  }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(aux), t.a.bk, 0, t.a.bmean, t.a.bvar, t.a.gamma_b,
                t.a.beta_b);
    fill_row_yx(const_cast<int*>(row_yx(aux)), static_cast<int64_t>(blockIdx.x) * kBM, t.a.M,
                t.a.H, t.a.W);
  }
  __device__ void produce(uint8_t* ah, uint8_t* al, uint8_t* bh, uint8_t* bl, int kb,
                          const uint8_t* aux) const {
    const LayerArgs<float>& a = t.a;
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;
    const int K = 9 * t.kp;
#pragma unroll
    for (int q = threadIdx.x; q < kBM * kBK / 8; q += kThreads) {
      int row, kc;
      kmajor_coords(q, row, kc);
      const int k0 = kb * kBK + kc;
      const int64_t p = m0 + row;
      float v[8];
      zero8(v);
      if (p < a.M && k0 < K) {
        const int tap = k0 / t.kp, o0 = k0 - tap * t.kp;
        int64_t src;  // dx[p] = sum_tap dy[p - d_tap] W[tap]
        if (o0 < a.k && neighbour(p, row_yx(aux)[row], a.H, a.W, 1 - tap / 3, 1 - tap % 3, src))
          load8(a.acc + src * a.Ca + a.c + o0, a.k - o0, t.vec, v);
      }
      put8<false>(ah, al, Tile<kBM>::kmajor_chunk(row, kc), v);
    }
#pragma unroll
    for (int q = threadIdx.x; q < BN * kBK / 8; q += kThreads) {
      int j, kc;
      kmajor_coords(q, j, kc);
      const int k0 = kb * kBK + kc;
      float v[8];
      zero8(v);
      if (j < a.bk && k0 < K) {
        const int tap = k0 / t.kp, o0 = k0 - tap * t.kp;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (o0 + i < a.k) v[i] = __ldg(a.w2 + (static_cast<int64_t>(o0 + i) * a.bk + j) * 9 + tap);
      }
      put8<false>(bh, bl, Tile<BN>::kmajor_chunk(j, kc), v);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t* aux,
                           float (&s1)[8], float (&s2)[8]) const {
    const LayerArgs<float>& a = t.a;
    const BnFwd* bn = reinterpret_cast<const BnFwd*>(aux);
    const int64_t p = static_cast<int64_t>(blockIdx.x) * kBM + row;
    const int nv = p < a.M ? a.bk - col0 : 0;
    float zv[8], g[8];
    if (nv > 0) load8(a.z + p * a.bk + col0, nv, (a.bk & 3) == 0, zv);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < nv) {
        const BnFwd b = bn[col0 + i];
        g[i] = relu_mask_ref(b, zv[i]) ? v[i] : 0.f;  // relu_backward by act_b
        s1[i] = g[i];
        s2[i] = g[i] * ((zv[i] - b.mean) * b.inv);
      } else {
        g[i] = 0.f;
        s1[i] = 0.f;
        s2[i] = 0.f;
      }
    }
    if (nv > 0) store8(a.g0 + p * a.bk + col0, nv, (a.bk & 3) == 0, g);
  }
  __device__ void col_sums(int c, double s1, double s2) const {
    if (c < t.a.bk) t.a.part[static_cast<int64_t>(blockIdx.x) * t.a.bk + c] = make_double2(s1, s2);
  }
};

// ---- backward 1x1 dgrad: t2 = relu'(act_a) * (t1 . W1), bf16, N tiled --------------
template <int BN_>
struct Tc1x1Dgrad {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = false, kColSums = true, kF16 = false;
  static constexpr int kAMN = 0, kBMN = 1;
  TcArgs t;
  __device__ int num_kb() const { return (t.a.bk + kBK - 1) / kBK; }
  __device__ const BnFwd* tile_a(const uint8_t* aux) const {
    return reinterpret_cast<const BnFwd*>(aux + ((sizeof(BnBwd) * t.a.bk + 15) / 16) * 16);
  }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_bwd(reinterpret_cast<BnBwd*>(aux), t.a);
    const int n0 = blockIdx.y * BN;
    const int cnt = t.a.c - n0 < BN ? t.a.c - n0 : BN;
    fill_bn_fwd(const_cast<BnFwd*>(tile_a(aux)), cnt, n0, t.a.amean, t.a.avar, t.a.gamma_a,
                t.a.beta_a);
  }
  __device__ void produce(uint8_t* ah, uint8_t* al, uint8_t* bh, uint8_t* bl, int kb,
                          const uint8_t* aux) const {
    const LayerArgs<float>& a = t.a;
    const BnBwd* bb = reinterpret_cast<const BnBwd*>(aux);
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kBM;
#pragma unroll
    for (int q = threadIdx.x; q < kBM * kBK / 8; q += kThreads) {
      int row, kc;
      kmajor_coords(q, row, kc);
      const int j0 = kb * kBK + kc;
      const int64_t p = m0 + row;
      float v[8];
      const int nv = a.bk - j0;
      if (p < a.M && nv > 0) {
        float zv[8];
        load8(a.g0 + p * a.bk + j0, nv, (a.bk & 3) == 0, v);
        load8(a.z + p * a.bk + j0, nv, (a.bk & 3) == 0, zv);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = i < nv ? bnb_t1(bb[j0 + i], v[i], zv[i]) : 0.f;
      } else {
        zero8(v);
      }
      put8<false>(ah, al, Tile<kBM>::kmajor_chunk(row, kc), v);
    }
    // B(i, j) = W1[j][i]: MN-major, 8 consecutive i of row j per chunk
    const int n0 = blockIdx.y * BN;
#pragma unroll
    for (int q = threadIdx.x; q < BN * kBK / 8; q += kThreads) {
      int rg, kr;
      mnmajor_coords<BN>(q, rg, kr);
      const int j = kb * kBK + kr;
      const int i0 = n0 + rg;
      float v[8];
      if (j < a.bk && i0 < a.c) load8(a.w1 + static_cast<int64_t>(j) * a.c + i0, a.c - i0, false, v);
      else zero8(v);
      put8<false>(bh, bl, Tile<BN>::mnmajor_chunk(rg, kr), v);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t* aux,
                           float (&s1)[8], float (&s2)[8]) const {
    const LayerArgs<float>& a = t.a;
    const BnFwd* bn = tile_a(aux);
    const int64_t p = static_cast<int64_t>(blockIdx.x) * kBM + row;
    const int i0 = blockIdx.y * BN + col0;
    const int nv = p < a.M ? a.c - i0 : 0;
    float x[8], g[8];
    if (nv > 0) load8(a.feat + p * a.C + i0, nv, t.vec, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < nv) {
        const BnFwd b = bn[col0 + i];
        g[i] = relu_mask_ref(b, x[i]) ? v[i] : 0.f;  // relu_backward by act_a
        s1[i] = g[i];
        s2[i] = g[i] * ((x[i] - b.mean) * b.inv);
      } else {
        g[i] = 0.f;
        s1[i] = 0.f;
        s2[i] = 0.f;
      }
    }
    if (nv > 0) store8(a.g1 + p * a.cg + i0, nv, (a.cg & 3) == 0, g);
  }
  __device__ void col_sums(int c, double s1, double s2) const {
    const int i = blockIdx.y * BN + c;
    if (i < t.a.c) t.a.part[static_cast<int64_t>(blockIdx.x) * t.a.c + i] = make_double2(s1, s2);
  }
};

// ---- backward 1x1 wgrad: dW1^T[i][j] = sum_p act_a[p,i] t1[p,j], split over pixels -
template <int BN_>
struct Tc1x1Wgrad {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = false, kColSums = false, kF16 = false;
  static constexpr int kAMN = 1, kBMN = 1;
  TcArgs t;
  __device__ int64_t kbeg() const { return static_cast<int64_t>(blockIdx.z) * t.a.kchunk; }
  __device__ int num_kb() const {
    const int64_t e = kbeg() + t.a.kchunk < t.a.M ? kbeg() + t.a.kchunk : t.a.M;
    return static_cast<int>((e - kbeg() + kBK - 1) / kBK);
  }
  __device__ int64_t kend() const {
    return kbeg() + t.a.kchunk < t.a.M ? kbeg() + t.a.kchunk : t.a.M;
  }
  __device__ const BnFwd* tile_a(const uint8_t* aux) const {
    return reinterpret_cast<const BnFwd*>(aux + ((sizeof(BnBwd) * t.a.bk + 15) / 16) * 16);
  }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_bwd(reinterpret_cast<BnBwd*>(aux), t.a);
    const int m0 = blockIdx.x * kBM;
    const int cnt = t.a.c - m0 < kBM ? t.a.c - m0 : kBM;
    fill_bn_fwd(const_cast<BnFwd*>(tile_a(aux)), cnt, m0, t.a.amean, t.a.avar, t.a.gamma_a,
                t.a.beta_a);
  }
  __device__ void produce(uint8_t* ah, uint8_t* al, uint8_t* bh, uint8_t* bl, int kb,
                          const uint8_t* aux) const {
    const LayerArgs<float>& a = t.a;
    const BnFwd* bn = tile_a(aux);
    const BnBwd* bb = reinterpret_cast<const BnBwd*>(aux);
    const int m0 = blockIdx.x * kBM;
    const int64_t pk = kbeg() + static_cast<int64_t>(kb) * kBK, pe = kend();
    // A: rows = channels i (MN-major), K = pixels
#pragma unroll
    for (int q = threadIdx.x; q < kBM * kBK / 8; q += kThreads) {
      int rg, kr;
      mnmajor_coords<kBM>(q, rg, kr);
      const int64_t p = pk + kr;
      const int i0 = m0 + rg;
      float v[8];
      const int nv = a.c - i0;
      if (p < pe && nv > 0) {
        load8(a.feat + p * a.C + i0, nv, t.vec, v);
        bnrelu8(bn, rg, nv, v);
      } else {
        zero8(v);
      }
      put8<false>(ah, al, Tile<kBM>::mnmajor_chunk(rg, kr), v);
    }
    // B: rows = bk channels j (MN-major), K = pixels, t1 recomputed
#pragma unroll
    for (int q = threadIdx.x; q < BN * kBK / 8; q += kThreads) {
      int rg, kr;
      mnmajor_coords<BN>(q, rg, kr);
      const int64_t p = pk + kr;
      float v[8];
      const int nv = a.bk - rg;
      if (p < pe && nv > 0) {
        float zv[8];
        load8(a.g0 + p * a.bk + rg, nv, (a.bk & 3) == 0, v);
        load8(a.z + p * a.bk + rg, nv, (a.bk & 3) == 0, zv);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = i < nv ? bnb_t1(bb[rg + i], v[i], zv[i]) : 0.f;
      } else {
        zero8(v);
      }
      put8<false>(bh, bl, Tile<BN>::mnmajor_chunk(rg, kr), v);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&)[8],
                           float (&)[8]) const {
    const LayerArgs<float>& a = t.a;
    const int i = blockIdx.x * kBM + row;
    const int nv = i < a.c ? a.bk - col0 : 0;
    if (nv > 0)
      store8(a.wpart + (static_cast<int64_t>(blockIdx.z) * a.c + i) * a.bk + col0, nv,
             (a.bk & 3) == 0, v);
  }
  __device__ void col_sums(int, double, double) const {}
};

// ---- backward 3x3 wgrad: dW2[(tap,j)][o] = sum_p act_b[p+d_tap, j] dY[p, o] --------
template <int BN_>
struct Tc3x3Wgrad {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = false, kColSums = false, kF16 = false;
  static constexpr int kAMN = 1, kBMN = 1;
  TcArgs t;
  __device__ int64_t kbeg() const { return static_cast<int64_t>(blockIdx.z) * t.a.kchunk; }
  __device__ int64_t kend() const {
    return kbeg() + t.a.kchunk < t.a.M ? kbeg() + t.a.kchunk : t.a.M;
  }
  __device__ int num_kb() const { return static_cast<int>((kend() - kbeg() + kBK - 1) / kBK); }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(aux), t.a.bk, 0, t.a.bmean, t.a.bvar, t.a.gamma_b,
                t.a.beta_b);
  }
  __device__ void produce(uint8_t* ah, uint8_t* al, uint8_t* bh, uint8_t* bl, int kb,
                          const uint8_t* aux) const {
    const LayerArgs<float>& a = t.a;
    const BnFwd* bn = reinterpret_cast<const BnFwd*>(aux);
    const int m0 = blockIdx.x * kBM;
    const int R = 9 * a.bk;
    const int64_t pk = kbeg() + static_cast<int64_t>(kb) * kBK, pe = kend();
#pragma unroll
    for (int q = threadIdx.x; q < kBM * kBK / 8; q += kThreads) {
      int rg, kr;
      mnmajor_coords<kBM>(q, rg, kr);
      const int64_t p = pk + kr;
      const int r0 = m0 + rg;
      float v[8];
      zero8(v);
      if (p < pe && r0 < R) {
        const int tap = r0 / a.bk, j0 = r0 - tap * a.bk;
        int64_t nb;
        if (shifted(p, a.H, a.W, tap / 3 - 1, tap % 3 - 1, nb)) {
          load8(a.z + nb * a.bk + j0, 8, (a.bk & 3) == 0, v);
          bnrelu8(bn, j0, 8, v);
        }
      }
      put8<false>(ah, al, Tile<kBM>::mnmajor_chunk(rg, kr), v);
    }
#pragma unroll
    for (int q = threadIdx.x; q < BN * kBK / 8; q += kThreads) {
      int rg, kr;
      mnmajor_coords<BN>(q, rg, kr);
      const int64_t p = pk + kr;
      float v[8];
      if (p < pe && rg < a.k) load8(a.acc + p * a.Ca + a.c + rg, a.k - rg, t.vec, v);
      else zero8(v);
      put8<false>(bh, bl, Tile<BN>::mnmajor_chunk(rg, kr), v);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&)[8],
                           float (&)[8]) const {
    const LayerArgs<float>& a = t.a;
    const int r = blockIdx.x * kBM + row;
    const int nv = r < 9 * a.bk ? a.k - col0 : 0;
    if (nv > 0)
      store8(a.wpart + (static_cast<int64_t>(blockIdx.z) * 9 * a.bk + r) * a.k + col0, nv, false, v);
  }
  __device__ void col_sums(int, double, double) const {}
};

}  // namespace tc
}  // namespace dpb
