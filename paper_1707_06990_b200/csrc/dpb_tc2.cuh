// Persistent, warp-specialised tcgen05 engine fed by TMA (engine v2).
//
// One CTA per SM loops over output tiles (tile = blockIdx.x, += gridDim.x).
// Warp roles (448 threads):
//   warp 0        TMA: streams the op's raw fp32 tiles (2D tensor maps,
//                 128-byte swizzle) into a ring of kNR raw stages
//   warp 1        MMA: one elected thread issues tcgen05.mma per operand
//                 stage into one of two TMEM accumulators, commits stages
//                 back to the transform warps and finished accumulators to
//                 the epilogue
//   warps 2-5     epilogue: tcgen05.ld the accumulator of tile i while the
//                 MMA already accumulates tile i+1 into the other buffer
//   warps 6-13    transform: raw fp32 smem -> fused BN/ReLU (or BN backward)
//                 -> bf16 (hi/lo for the bf16x3 forward) UMMA operand stages
// Every hand-off is an mbarrier (TMA tx-count, tcgen05.commit, or warp
// arrivals), so HBM loads, operand transforms, MMAs and epilogues of
// different tiles overlap — the per-tile latency chain of the v1 engine is
// gone.  Deterministic: each tile's column reductions are written to its own
// partial slot.
#pragma once

#include <cuda.h>

#include "dpb_simt.cuh"
#include "dpb_tc.cuh"
#include "dpb_tc_ops.cuh"

namespace dpb {
namespace tc2 {

using tc::kBK;
using tc::kBM;

constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kNumEpiWarps = 4;
constexpr int kXfWarp0 = 6, kNumXfWarps = 8;
constexpr int kXfThreads = 32 * kNumXfWarps;
constexpr int kThreads = 32 * (kXfWarp0 + kNumXfWarps);  // 448

using tc::bulk_load;
using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::named_sync;
using tc::prefetch_tmap;
using tc::tma_load_2d;

// Raw fp32 tile loaded by TMA with 128-byte swizzle: box = 32 channels x rows.
// Element (row, ch) of box b lives at b*box_bytes + row*128 + (((ch/4) ^ (row%8))*16) + (ch%4)*4.
// Reads 8 consecutive channels (two 16-byte chunks) starting at ch (ch % 8 == 0).
__device__ __forceinline__ void raw_read8(const uint8_t* box, int row, int ch, float (&v)[8]) {
  const int c4 = ch >> 2;
  const float4 a = *reinterpret_cast<const float4*>(box + row * 128 + (((c4) ^ (row & 7)) << 4));
  const float4 b = *reinterpret_cast<const float4*>(box + row * 128 + (((c4 + 1) ^ (row & 7)) << 4));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// Warp reduction of 8 columns x 32 rows in 9 shuffles (transpose-reduce): on
// return lane L holds the full column sum of column (L >> 2) & 7 in v[0].
__device__ __forceinline__ float warp_colsum8(float (&v)[8], int lane) {
  // step 1: exchange halves of the 8 values with lane ^ 16
  {
    const bool up = lane & 16;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float send = up ? v[i] : v[i + 4];
      const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
      v[i] = (up ? v[i + 4] : v[i]) + recv;
    }
  }
  // lanes with bit 4 set now hold columns 4..7 in v[0..3], others 0..3
  {
    const bool up = lane & 8;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float send = up ? v[i] : v[i + 2];
      const float recv = __shfl_xor_sync(0xffffffffu, send, 8);
      v[i] = (up ? v[i + 2] : v[i]) + recv;
    }
  }
  {
    const bool up = lane & 4;
    const float send = up ? v[0] : v[1];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 4);
    v[0] = (up ? v[1] : v[0]) + recv;
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  // column held by this lane: bit4 -> +4, bit3 -> +2, bit2 -> +1
  return v[0];
}
__device__ __forceinline__ int colsum8_column(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}

// ---- the engine ------------------------------------------------------------------
// Op interface:
//   static constexpr int BN, kTmemCols, kNR, kNS, kRawBytes, kOpBytes; bool kColSums
//   int num_tiles() const;  int num_kb(int tile) const;  void prefetch() const;
//   void prologue(uint8_t* aux) const;                         all threads
//   uint32_t raw_bytes(int tile, int kb) const;                bytes the stage's copies land
//   void tma(int tile, int kb, uint32_t raw, uint64_t* bar) const;   one thread
//   static constexpr bool kMmaReadsRaw;                         MMA reads pre-tiled B from
//                                                              the raw stage
//   void transform(int tile, int kb, const uint8_t* raw, uint8_t* opnd,
//                  const uint8_t* aux, int xt) const;          256 transform threads
//   void mma(uint32_t opnd, uint32_t raw, uint32_t aux, uint32_t tmem, int kb) const;
//   void epilogue(int tile, int row, int col0, const float (&v)[8], const uint8_t* aux,
//                 float (&s1)[8], float (&s2)[8]) const;       128 epilogue threads
//   void col_sums(int tile, int col, double s1, double s2) const;
template <class Op>
__global__ void __launch_bounds__(kThreads, 1) tc2_kernel(const __grid_constant__ Op op) {
  constexpr int NR = Op::kNR, NS = Op::kNS, BN = Op::BN;
  constexpr uint32_t TC = tc::TmemCols<Op::kTmemCols>::value;
  static_assert(2 * TC <= 512, "two TMEM accumulators");
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  // TMA 128-byte swizzle needs 1024-byte aligned destinations
  uint8_t* smem = smem_dyn + ((1024 - (tc::smem_u32(smem_dyn) & 1023)) & 1023);
  __shared__ uint64_t raw_full[NR], raw_empty[NR], op_full[NS], op_empty[NS];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float red[2][4][BN];

  uint8_t* raw_ring = smem;
  uint8_t* op_ring = smem + NR * Op::kRawBytes;
  uint8_t* aux = op_ring + NS * Op::kOpBytes;  // op tables; resident B images first

  const int tid = threadIdx.x;
  const int warp = tid / 32, lane = tid % 32;
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) {
      tc::mbar_init(&raw_full[i], 1);
      tc::mbar_init(&raw_empty[i], kNumXfWarps + (Op::kMmaReadsRaw ? 1 : 0));
    }
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&op_full[i], kNumXfWarps);
      tc::mbar_init(&op_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], kNumEpiWarps);
    }
    tc::fence_barrier_init();
  }
  if (warp == kMmaWarp) tc::tmem_alloc<2 * TC>(&tmem_base);
  op.prologue(aux);
  tc::fence_proxy_async();  // resident operand images written by generic stores
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int ntiles = op.num_tiles();

  if (warp == kTmaWarp) {
    if (lane == 0) {
      op.prefetch();
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int kb = 0; kb < op.num_kb(tile); ++kb, ++it) {
          const int r = it % NR;
          tc::mbar_wait(&raw_empty[r], ((it / NR) & 1) ^ 1);
          mbar_expect_tx(&raw_full[r], op.raw_bytes(tile, kb));
          op.tma(tile, kb, tc::smem_u32(raw_ring + r * Op::kRawBytes), &raw_full[r]);
        }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      int it = 0, at = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++at) {
        const int a = at & 1;
        tc::mbar_wait(&acc_empty[a], ((at >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        for (int kb = 0; kb < op.num_kb(tile); ++kb, ++it) {
          const int s = it % NS, r = it % NR;
          tc::mbar_wait(&op_full[s], (it / NS) & 1);
          tc::tc_fence_after();
          op.mma(tc::smem_u32(op_ring + s * Op::kOpBytes), tc::smem_u32(raw_ring + r * Op::kRawBytes),
                 tc::smem_u32(aux), tmem + a * TC, kb);
          tc::mma_commit(&op_empty[s]);
          if constexpr (Op::kMmaReadsRaw) tc::mma_commit(&raw_empty[r]);
        }
        tc::mma_commit(&acc_full[a]);
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kNumEpiWarps) {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int et = tid - kEpiWarp0 * 32;  // 0..127
    int at = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++at) {
      const int a = at & 1;
      tc::mbar_wait(&acc_full[a], (at >> 1) & 1);
      tc::tc_fence_after();
      for (int cc = 0; cc < Op::kTmemCols / 8; ++cc) {
        float v[8];
        tc::tmem_ld8(tmem + a * TC + (static_cast<uint32_t>(quarter * 32) << 16) + cc * 8, v);
        float s1[8], s2[8];
        op.epilogue(tile, row, cc * 8, v, aux, s1, s2);
        if constexpr (Op::kColSums) {
          const float x = warp_colsum8(s1, lane);
          const float y = warp_colsum8(s2, lane);
          if ((lane & 3) == 0) {
            const int col = cc * 8 + colsum8_column(lane);
            red[0][quarter][col] = x;
            red[1][quarter][col] = y;
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
      if constexpr (Op::kColSums) {
        named_sync(1, 32 * kNumEpiWarps);
        for (int c = et; c < BN; c += 32 * kNumEpiWarps) {
          const double x = static_cast<double>(red[0][0][c]) + red[0][1][c] + red[0][2][c] + red[0][3][c];
          const double y = static_cast<double>(red[1][0][c]) + red[1][1][c] + red[1][2][c] + red[1][3][c];
          op.col_sums(tile, c, x, y);
        }
        named_sync(1, 32 * kNumEpiWarps);
      }
    }
  } else {
    const int xt = tid - kXfWarp0 * 32;  // 0..255
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < op.num_kb(tile); ++kb, ++it) {
        const int r = it % NR, s = it % NS;
        tc::mbar_wait(&raw_full[r], (it / NR) & 1);
        tc::mbar_wait(&op_empty[s], ((it / NS) & 1) ^ 1);
        op.transform(tile, kb, raw_ring + r * Op::kRawBytes, op_ring + s * Op::kOpBytes, aux, xt);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&op_full[s]);
          mbar_arrive(&raw_empty[r]);
        }
      }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    tc::tmem_dealloc<2 * TC>(tmem);
  }
}

// ---- 1x1 forward: z = relu(bn_a(x)) . W1^T (bf16x3) ---------------------------------
// raw stage: x rows [m0, m0+128) x channels [64 kb, 64 kb + 64) as one or two
// 32-channel TMA boxes (only the boxes that hold channels < c).  W1's
// pre-tiled bf16 hi | lo operand tiles are either resident in shared memory
// for the whole persistent CTA (RES: copied once in the prologue) or
// streamed per K block into the raw stage by a 1D bulk copy (large c).
// Operand stage: A hi | A lo.
template <int BN_, bool RES>
struct Fwd1x1 {
  static constexpr int BN = BN_;
  static constexpr int kTmemCols = BN;
  static constexpr bool kColSums = true;
  static constexpr bool kMmaReadsRaw = !RES;
  static constexpr int kBox = 32 * kBM * 4;                    // 16 KB
  static constexpr int kBBytes = tc::Tile<BN>::kBytes;
  static constexpr int kRawBytes = 2 * kBox + (RES ? 0 : 2 * kBBytes);
  static constexpr int kNR = RES ? 3 : (BN <= 64 ? 3 : 2);
  static constexpr int kABytes = tc::Tile<kBM>::kBytes;         // 16 KB
  static constexpr int kOpBytes = 2 * kABytes;
  static constexpr int kNS = 2;
  CUtensorMap xmap;        // feat [M][C] fp32, box {32, 128}, swizzle 128B
  LayerArgs<float> a;
  const uint8_t* w1t;      // pre-tiled W1: per K block, hi tile | lo tile (Tile<BN> K-major)

  __device__ void prefetch() const { prefetch_tmap(&xmap); }
  __device__ int num_tiles() const { return static_cast<int>((a.M + kBM - 1) / kBM); }
  __device__ int num_kb(int) const { return (a.c + kBK - 1) / kBK; }
  __device__ int boxes(int kb) const { return a.c - kb * kBK > 32 ? 2 : 1; }
  __device__ uint32_t raw_bytes(int, int kb) const {
    return boxes(kb) * kBox + (RES ? 0 : 2 * kBBytes);
  }
  __device__ uint32_t b_all() const { return static_cast<uint32_t>(num_kb(0) * 2 * kBBytes); }
  __device__ const BnFwd* bn_table(const uint8_t* aux) const {
    return reinterpret_cast<const BnFwd*>(aux + (RES ? b_all() : 0));
  }
  __device__ void prologue(uint8_t* aux) const {
    if (RES) {
      const uint4* src = reinterpret_cast<const uint4*>(w1t);
      uint4* dst = reinterpret_cast<uint4*>(aux);
      for (int q = threadIdx.x; q < static_cast<int>(b_all() / 16); q += kThreads) dst[q] = __ldg(src + q);
    }
    fill_bn_fwd(const_cast<BnFwd*>(bn_table(aux)), a.c, 0, a.amean, a.avar, a.gamma_a, a.beta_a);
  }
  __device__ void tma(int tile, int kb, uint32_t raw, uint64_t* bar) const {
    tma_load_2d(raw, &xmap, kb * kBK, tile * kBM, bar);
    if (boxes(kb) == 2) tma_load_2d(raw + kBox, &xmap, kb * kBK + 32, tile * kBM, bar);
    if (!RES) bulk_load(raw + 2 * kBox, w1t + static_cast<int64_t>(kb) * 2 * kBBytes, 2 * kBBytes, bar);
  }
  __device__ void transform(int, int kb, const uint8_t* raw, uint8_t* op, const uint8_t* aux,
                            int xt) const {
    const BnFwd* bn = bn_table(aux);
    uint8_t* ah = op;
    uint8_t* al = op + kABytes;
    // every chunk of this thread covers the same 8 channels (kmajor_coords):
    // BN as one FMA per element with per-stage register coefficients
    int row0, kc;
    tc::kmajor_coords(xt, row0, kc);
    const int ch0 = kb * kBK + kc;
    float sc[8], sh[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (ch0 + i < a.c) {
        const BnFwd b = bn[ch0 + i];
        sc[i] = b.scale;
        sh[i] = fmaf(-b.mean, b.scale, b.beta);
      } else {
        sc[i] = 0.f;  // channels past c contribute zero
        sh[i] = 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < kBM * kBK / 8 / kXfThreads; ++i) {
      const int row = row0 + i * (kXfThreads / 8);
      float v[8];
      if (ch0 < a.c) {
        raw_read8(raw + (kc >> 5) * kBox, row, kc & 31, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = fmaxf(fmaf(v[e], sc[e], sh[e]), 0.f);
      } else {
        tc::zero8(v);
      }
      uint4 h, l;
      tc::split8_fast(v, h, l);
      const uint32_t off = tc::Tile<kBM>::kmajor_chunk(row, kc);
      tc::st_shared16(ah, off, h);
      tc::st_shared16(al, off, l);
    }
  }
  __device__ void mma(uint32_t op, uint32_t raw, uint32_t aux, uint32_t tmem, int kb) const {
    constexpr uint32_t idesc = tc::make_idesc(BN, 0, 0);
    const uint32_t ah = op, al = op + kABytes;
    const uint32_t bh = RES ? aux + kb * 2 * kBBytes : raw + 2 * kBox, bl = bh + kBBytes;
#pragma unroll
    for (int k16 = 0; k16 < kBK / 16; ++k16) {
      const uint32_t acc = (kb | k16) ? 1u : 0u;
      tc::mma_bf16(tmem, tc::Tile<kBM>::desc(ah, k16), tc::Tile<BN>::desc(bh, k16), idesc, acc);
      tc::mma_bf16(tmem, tc::Tile<kBM>::desc(ah, k16), tc::Tile<BN>::desc(bl, k16), idesc, 1u);
      tc::mma_bf16(tmem, tc::Tile<kBM>::desc(al, k16), tc::Tile<BN>::desc(bh, k16), idesc, 1u);
    }
  }
  __device__ void epilogue(int tile, int row, int col0, const float (&v)[8], const uint8_t*,
                           float (&s1)[8], float (&s2)[8]) const {
    const int64_t p = static_cast<int64_t>(tile) * kBM + row;
    const int nv = p < a.M ? a.bk - col0 : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = i < nv;
      s1[i] = ok ? v[i] : 0.f;
      s2[i] = ok ? v[i] * v[i] : 0.f;
    }
    if (nv > 0) tc::store8(a.z + p * a.bk + col0, nv, (a.bk & 3) == 0, v);
  }
  __device__ void col_sums(int tile, int c, double s1, double s2) const {
    if (c < a.bk) a.part[static_cast<int64_t>(tile) * a.bk + c] = make_double2(s1, s2);
  }
};

// All layers of a block in one launch: blockIdx.y = layer.
template <int BN>
__global__ void k_pretile_w1_all(const float* __restrict__ params, int c0, int k, int bk, int m,
                                 uint8_t* __restrict__ out) {
  const int l = blockIdx.y;
  int64_t poff = 0, toff = 0;
  for (int j = 0; j < l; ++j) {
    const int cj = c0 + j * k;
    poff += 2LL * cj + static_cast<int64_t>(bk) * cj + 2LL * bk + 9LL * k * bk;
    toff += static_cast<int64_t>((cj + kBK - 1) / kBK) * 2 * tc::Tile<BN>::kBytes;
  }
  const int c = c0 + l * k;
  const float* w1 = params + poff + 2 * c;
  const int nkb = (c + kBK - 1) / kBK;
  const int chunks = BN * kBK / 8;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nkb * chunks; q += gridDim.x * blockDim.x) {
    const int kb = q / chunks, qq = q - kb * chunks;
    const int row = qq / 8, kc = (qq % 8) * 8;
    const int i0 = kb * kBK + kc;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = (row < bk && i0 + i < c) ? w1[static_cast<int64_t>(row) * c + i0 + i] : 0.f;
    uint4 h, lo;
    tc::split8(v, h, lo);
    uint8_t* t = out + toff + static_cast<int64_t>(kb) * 2 * tc::Tile<BN>::kBytes;
    const uint32_t off = tc::Tile<BN>::kmajor_chunk(row, kc);
    *reinterpret_cast<uint4*>(t + off) = h;
    *reinterpret_cast<uint4*>(t + tc::Tile<BN>::kBytes + off) = lo;
  }
}

}  // namespace tc2
}  // namespace dpb
