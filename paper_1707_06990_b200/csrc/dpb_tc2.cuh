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
//   warps 2-9     epilogue: tcgen05.ld the accumulator of tile i while the
//                 MMA already accumulates tile i+1 into the other buffer; two
//                 groups of four warps (one per TMEM lane quarter) take
//                 alternate 32-column groups, one 32-column TMEM load each
//   warps 10-17   transform: raw fp32 smem -> fused BN/ReLU (or BN backward)
//                 -> bf16 (hi/lo for the bf16x3 forward) UMMA operand stages
//   warp 18       epilogue loads: streams the tiles the epilogue reads (e.g.
//                 the features whose ReLU mask the backward applies) into a
//                 ring of kNE boxes, one tile ahead of the epilogue
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

constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2;

// Warp roles of an op: kEpiWarps epilogue warps (groups of four, one warp per
// TMEM lane quarter; groups take alternate 32-column boxes), kXfWarps
// transform warps, then the epilogue-load warp.
template <class Op>
struct Roles {
  static constexpr int kEpi = Op::kEpiWarps;
  static constexpr int kGroups = kEpi / 4;
  static constexpr int kXf = Op::kXfWarps;
  static constexpr int kXfWarp0 = kEpiWarp0 + kEpi;
  static constexpr int kLoadWarp = kXfWarp0 + kXf;
  static constexpr int kThreads = 32 * (kLoadWarp + 1);
  static_assert(kEpi % 4 == 0 && kEpi >= 4, "epilogue warps come in groups of four");
};

using tc::bulk_load;
using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::named_sync;
using tc::prefetch_tmap;
using tc::tma_load_2d;

// Raw fp32 tile loaded by TMA with 128-byte swizzle: box = 32 channels x rows.
// Element (row, ch) of box b lives at b*box_bytes + row*128 + (((ch/4) ^ (row%8))*16) + (ch%4)*4.
// Reads 8 consecutive channels (two 16-byte chunks) starting at ch (ch % 8 == 0);
// raw_write8 writes them back in place (the epilogue's TMA-store staging).
__device__ __forceinline__ void raw_read8(const uint8_t* box, int row, int ch, float (&v)[8]) {
  const int c4 = ch >> 2;
  const float4 a = *reinterpret_cast<const float4*>(box + row * 128 + (((c4) ^ (row & 7)) << 4));
  const float4 b = *reinterpret_cast<const float4*>(box + row * 128 + (((c4 + 1) ^ (row & 7)) << 4));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void raw_write8(uint8_t* box, int row, int ch, const float (&v)[8]) {
  const int c4 = ch >> 2;
  *reinterpret_cast<float4*>(box + row * 128 + (((c4) ^ (row & 7)) << 4)) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(box + row * 128 + (((c4 + 1) ^ (row & 7)) << 4)) = make_float4(v[4], v[5], v[6], v[7]);
}

// BN_a tables of the backward kernels as one float4 per channel (one 16-byte
// shared load per element instead of a 20-byte BnFwd's scalar loads):
//   mask form  {mean, inv, gamma, beta}   relu_mask_ref's exact expression
//   apply form {mean, gamma*inv, beta, 0}  bn_relu's fmaf(x - mean, scale, beta)
__device__ __forceinline__ void fill_bn_mask4(float4* t, int count, int first, const float* mean,
                                              const float* var, const float* gamma, const float* beta) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const int ch = first + i;
    t[i] = make_float4(mean[ch], bn_inv(var[ch]), gamma[ch], beta[ch]);
  }
}
__device__ __forceinline__ void fill_bn_apply4(float4* t, int count, int first, const float* mean,
                                               const float* var, const float* gamma, const float* beta) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const int ch = first + i;
    t[i] = make_float4(mean[ch], gamma[ch] * bn_inv(var[ch]), beta[ch], 0.f);
  }
}
__device__ __forceinline__ bool relu_mask4(const float4& b, float x) {  // == relu_mask_ref
  const float t = __fmul_rn(__fmul_rn(b.z, __fsub_rn(x, b.x)), b.y);
  return __fadd_rn(t, b.w) > 0.f;
}
using tc::colsum8_column;
using tc::warp_colsum8;

// Debug-only phase clocks (dpb_debug_tc2_clocks): when g_tc2_dbg_c equals the
// launch's layer width a.c, CTA x (< 148, column tile 0) stamps %globaltimer (ns) at
//   [0] start [1] prologue done [2+t] TMA first load of tile t
//   [6+t] transform of tile t done [10+t] MMA of tile t committed
//   [14+t] epilogue of tile t starts [18+t] ends [22] exit   (t < 4)
__device__ __forceinline__ long long dbg_now() {  // ns, synchronised across SMs
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<long long>(t);
}
// [23] / [24]: epi_full wait, warp 2 / warp 6; [25] / [26]: transform warp 0 wait for
// raw_full / op_empty; [27]: TMA thread wait for raw_empty (ns summed over the launch)
__device__ long long g_tc2_clock[148][28];
__device__ int g_tc2_dbg_c;

// ---- the engine ------------------------------------------------------------------
// Op interface:
//   static constexpr int BN, kTmemCols, kNR, kNS, kRawBytes, kOpBytes; bool kColSums
//   static constexpr int kNE, kEpiBytes;                        epilogue ring (kNE = 0: none)
//   static constexpr bool kEpiStore;                            the epilogue rewrites each box in
//                                                              place and the load warp TMA-stores
//                                                              it (epi_store) before reusing it
//   int num_tiles() const;  int num_kb(int tile) const;  void prefetch() const;
//   int epi_chunks(int tile) const;                             8-column TMEM chunks
//   int epi_boxes(int tile) const;  void epi_tma(int tile, int b, uint32_t dst, uint64_t* bar) const;
//                                                              one box per 4 chunks (32 columns)
//   void epi_store(int tile, int b, uint32_t src) const;
//   void prologue_early(uint8_t* aux) const;                   all threads, before the
//                                                              grid-dependency wait
//   static constexpr bool kEarlyLoads;                          the first NR stages' TMA
//                                                              loads may precede the wait
//   void prologue(uint8_t* aux) const;                         all threads
//   uint32_t raw_bytes(int tile, int kb) const;                bytes the stage's copies land
//   void tma(int tile, int kb, uint32_t raw, uint64_t* bar) const;   one thread
//   static constexpr bool kMmaReadsRaw;                         MMA reads pre-tiled B from
//                                                              the raw stage
//   void transform(int tile, int kb, const uint8_t* raw, uint8_t* opnd,
//                  const uint8_t* aux, int xt) const;          256 transform threads
//   void mma(uint32_t opnd, uint32_t raw, uint32_t aux, uint32_t tmem, int kb) const;
//   void epilogue(int tile, int row, int col0, const float (&v)[8], const uint8_t* aux,
//                 uint8_t* ebox, float (&s1)[8], float (&s2)[8]) const;
//                                                              128 epilogue threads
//   void col_sums(int tile, int col, double s1, double s2) const;
template <class Op>
__global__ void __launch_bounds__(Roles<Op>::kThreads, 1) tc2_kernel(const __grid_constant__ Op op) {
  using R = Roles<Op>;
  // kInPlace ops transform each raw stage into its own UMMA operand (no operand
  // ring): stage r's op_full[r] hands it to the MMA, whose commit frees it.
  constexpr bool IP = Op::kInPlace;
  constexpr int NR = Op::kNR, NS = IP ? NR : Op::kNS, BN = Op::BN, NE = Op::kNE > 0 ? Op::kNE : 1;
  constexpr uint32_t TC = tc::TmemCols<Op::kTmemCols>::value;
  static_assert(2 * TC <= 512, "two TMEM accumulators");
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  // TMA 128-byte swizzle needs 1024-byte aligned destinations
  uint8_t* smem = smem_dyn + ((1024 - (tc::smem_u32(smem_dyn) & 1023)) & 1023);
  __shared__ uint64_t raw_full[NR], raw_empty[NR], op_full[NS], op_empty[NS];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint64_t epi_full[NE], epi_done[NE];
  __shared__ uint32_t tmem_base;
  __shared__ float red[2][4][BN];

  uint8_t* raw_ring = smem;
  uint8_t* op_ring = IP ? raw_ring : smem + NR * Op::kRawBytes;
  uint8_t* epi_ring = smem + NR * Op::kRawBytes + (IP ? 0 : NS * Op::kOpBytes);
  uint8_t* aux = epi_ring + Op::kNE * Op::kEpiBytes;  // op tables; resident B images first

  const int tid = threadIdx.x;
  const int warp = tid / 32, lane = tid % 32;
#ifdef DPB_PHASE_CLOCKS  // debug stamps (a global flag read at kernel entry)
  const bool dbg = Op::kColSums && g_tc2_dbg_c == op.a.c && blockIdx.x < 148 && blockIdx.y == 0;
#else
  constexpr bool dbg = false;
#endif
  long long* clk = g_tc2_clock[blockIdx.x < 148 ? blockIdx.x : 0];
  if (dbg && tid == 0) {
    clk[0] = dbg_now();
    clk[23] = clk[24] = clk[25] = clk[26] = clk[27] = 0;
  }
  if (tid == 0) {
    for (int i = 0; i < NR; ++i) {
      tc::mbar_init(&raw_full[i], 1);
      tc::mbar_init(&raw_empty[i], IP ? 1 : R::kXf + (Op::kMmaReadsRaw ? 1 : 0));
    }
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&op_full[i], R::kXf);
      tc::mbar_init(&op_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], R::kEpi);
    }
    for (int i = 0; i < NE; ++i) {
      tc::mbar_init(&epi_full[i], 1);
      tc::mbar_init(&epi_done[i], 4);  // one warp group per box
    }
    tc::fence_barrier_init();
  }
  if (warp == kMmaWarp) tc::tmem_alloc<2 * TC>(&tmem_base);
  // Before the grid-dependency wait a kernel may read what the launches two or
  // more back wrote (its predecessor passed its own wait before triggering this
  // launch): the resident weight images, tiled at the start of the pass.
  op.prologue_early(aux);
  // ... and, for ops whose TMA operands are at least two launches old
  // (kEarlyLoads), the first ring stages: the TMA thread initialised the
  // barriers itself, and the ring starts empty.
  int early = 0;
  if constexpr (Op::kEarlyLoads) {
    if (tid == 0) {
      op.prefetch();
      const int nt = op.num_tiles();
      for (int tile = blockIdx.x; tile < nt && early < NR; tile += gridDim.x)
        for (int kb = 0; kb < op.num_kb(tile) && early < NR; ++kb, ++early) {
          mbar_expect_tx(&raw_full[early], op.raw_bytes(tile, kb));
          op.tma(tile, kb, tc::smem_u32(raw_ring + early * Op::kRawBytes), &raw_full[early]);
        }
    }
  }
  pdl_enter();  // barrier init / TMEM alloc / weight copies above overlap the predecessor
  op.prologue(aux);
  tc::fence_proxy_async();  // resident operand images written by generic stores
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int ntiles = op.num_tiles();
  if (dbg && tid == 0) clk[1] = dbg_now();

  if (warp == kTmaWarp) {
    if (lane == 0) {
      op.prefetch();
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int kb = 0; kb < op.num_kb(tile); ++kb, ++it) {
          if (it < early) continue;  // issued before the wait
          const int r = it % NR;
          const long long w0 = dbg ? dbg_now() : 0;
          tc::mbar_wait(&raw_empty[r], ((it / NR) & 1) ^ 1);
          if (dbg) clk[27] += dbg_now() - w0;
          const int t = (tile - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x);
          if (dbg && kb == 0 && t < 4) clk[2 + t] = dbg_now();
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
          const uint8_t* opnd = IP ? raw_ring + r * Op::kRawBytes : op_ring + s * Op::kOpBytes;
          op.mma(tc::smem_u32(opnd), tc::smem_u32(raw_ring + r * Op::kRawBytes), tc::smem_u32(aux),
                 tmem + a * TC, kb);
          if constexpr (!IP) tc::mma_commit(&op_empty[s]);
          if constexpr (Op::kMmaReadsRaw || IP) tc::mma_commit(&raw_empty[r]);
        }
        tc::mma_commit(&acc_full[a]);
        if (dbg && at < 4) clk[10 + at] = dbg_now();
      }
    }
  } else if (warp >= kEpiWarp0 && warp < R::kXfWarp0) {
    const int quarter = warp & 3;                 // TMEM lanes this warp may read
    const int grp = (warp - kEpiWarp0) >> 2;      // first 32-column box of this warp's group
    const int row = quarter * 32 + lane;
    const int et = tid - kEpiWarp0 * 32;
    const bool sums = op.want_col_sums();  // (the split-K forward's come from its reduce pass)
    int at = 0, e0 = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++at) {
      const int a = at & 1;
      tc::mbar_wait(&acc_full[a], (at >> 1) & 1);
      tc::tc_fence_after();
      if (dbg && tid == kEpiWarp0 * 32 && at < 4) clk[14 + at] = dbg_now();
      const int nch = op.epi_chunks(tile);
      const int ngrp = (nch + 3) / 4;
      for (int gi = grp; gi < ngrp; gi += R::kGroups) {
        uint8_t* ebox = nullptr;
        const int e = e0 + gi;
        if constexpr (Op::kNE > 0) {
          const long long w0 = dbg ? dbg_now() : 0;
          tc::mbar_wait(&epi_full[e % NE], (e / NE) & 1);
          if (dbg && lane == 0 && (warp == kEpiWarp0 || warp == kEpiWarp0 + 4))
            clk[warp == kEpiWarp0 ? 23 : 24] += dbg_now() - w0;
          ebox = epi_ring + (e % NE) * Op::kEpiBytes;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
         if (gi * 4 + 2 * h < nch) {
          float v[16];
          tc::tmem_ld16(tmem + a * TC + (static_cast<uint32_t>(quarter * 32) << 16) + gi * 32 + h * 16, v);
#pragma unroll
          for (int q2 = 0; q2 < 2; ++q2) {
          const int q = 2 * h + q2;
          const int cc = gi * 4 + q;
          if (cc < nch) {
            float s1[8], s2[8];
            op.epilogue(tile, row, cc * 8, *reinterpret_cast<const float(*)[8]>(&v[q2 * 8]), aux, ebox,
                        s1, s2);
            if (Op::kColSums && sums) {
              const float x = warp_colsum8(s1, lane);
              const float y = warp_colsum8(s2, lane);
              if ((lane & 3) == 0) {
                const int col = cc * 8 + colsum8_column(lane);
                red[0][quarter][col] = x;
                red[1][quarter][col] = y;
              }
            }
          }
          }
         }
        }
        if constexpr (Op::kNE > 0) {  // box consumed (and rewritten) by this warp
          if constexpr (Op::kEpiStore) tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&epi_done[e % NE]);
        }
      }
      e0 += ngrp;
      if (dbg && tid == kEpiWarp0 * 32 && at < 4) clk[18 + at] = dbg_now();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
      if (Op::kColSums && sums) {
        named_sync(1, 32 * R::kEpi);
        for (int c = et; c < BN; c += 32 * R::kEpi) {
          const double x = static_cast<double>(red[0][0][c]) + red[0][1][c] + red[0][2][c] + red[0][3][c];
          const double y = static_cast<double>(red[1][0][c]) + red[1][1][c] + red[1][2][c] + red[1][3][c];
          op.col_sums(tile, c, x, y);
        }
        named_sync(1, 32 * R::kEpi);
      }
    }
  } else if (warp == R::kLoadWarp) {
    if constexpr (Op::kNE > 0) {
      if (lane == 0) {
        int e = 0;
        int slot_tile[NE] = {}, slot_box[NE] = {};  // box held by each slot (for the store)
        auto retire = [&](int s, int ee) {  // wait for box ee (slot s) to be processed
          tc::mbar_wait(&epi_done[s], (ee / NE) & 1);
          if constexpr (Op::kEpiStore) {
            op.epi_store(slot_tile[s], slot_box[s], tc::smem_u32(epi_ring + s * Op::kEpiBytes));
            tc::bulk_commit();
            tc::bulk_wait_read<0>();  // the slot may be overwritten once the store has read it
          }
        };
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
          for (int b = 0; b < op.epi_boxes(tile); ++b, ++e) {
            const int s = e % NE;
            if (e >= NE) retire(s, e - NE);
            mbar_expect_tx(&epi_full[s], Op::kEpiBytes);
            op.epi_tma(tile, b, tc::smem_u32(epi_ring + s * Op::kEpiBytes), &epi_full[s]);
            slot_tile[s] = tile;
            slot_box[s] = b;
          }
        for (int ee = e - NE > 0 ? e - NE : 0; ee < e; ++ee) retire(ee % NE, ee);
        if constexpr (Op::kEpiStore) tc::bulk_wait<0>();
      }
    }
  } else {
    const int xt = tid - R::kXfWarp0 * 32;  // 0 .. 32 * kXfWarps - 1
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < op.num_kb(tile); ++kb, ++it) {
        const int r = it % NR, s = it % NS;
        const long long w0 = dbg ? dbg_now() : 0;
        tc::mbar_wait(&raw_full[r], (it / NR) & 1);
        const long long w1 = dbg ? dbg_now() : 0;
        if constexpr (!IP) tc::mbar_wait(&op_empty[s], ((it / NS) & 1) ^ 1);
        if (dbg && tid == R::kXfWarp0 * 32) {
          clk[25] += w1 - w0;
          clk[26] += dbg_now() - w1;
        }
        uint8_t* rs = raw_ring + r * Op::kRawBytes;
        op.transform(tile, kb, rs, IP ? rs : op_ring + s * Op::kOpBytes, aux, xt);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&op_full[s]);
          if constexpr (!IP) mbar_arrive(&raw_empty[r]);
        }
        if (dbg && tid == R::kXfWarp0 * 32 && kb == op.num_kb(tile) - 1) {
          const int t = (tile - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x);
          if (t < 4) clk[6 + t] = dbg_now();
        }
      }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    tc::tmem_dealloc<2 * TC>(tmem);
  }
  if (dbg && tid == 0) clk[22] = dbg_now();
}

// ---- 1x1 forward: z = relu(bn_a(x)) . W1^T (bf16x3) ---------------------------------
// raw stage: x rows [m0, m0+128) x channels [64 kb, 64 kb + 64) as one or two
// 32-channel TMA boxes (only the boxes that hold channels < c).  W1's
// pre-tiled bf16 hi | lo operand tiles are either resident in shared memory
// for the whole persistent CTA (RES: copied once in the prologue) or
// streamed per K block into the raw stage by a 1D bulk copy (large c).
// Operand stage: A hi | A lo.
template <int BN_, bool RES, bool IP_ = false>
struct Fwd1x1 {
  static constexpr int BN = BN_;
  // IP_: in place — the operand A hi | A lo overwrites the stage's two fp32
  // boxes (32 KB each way), so the operand ring's shared memory buys a third
  // raw stage (streamed W1 only: one more stage of TMA latency in flight)
  static constexpr bool kInPlace = IP_;
  static constexpr int kTmemCols = BN;
  static constexpr bool kEarlyLoads = true;  // features / g0 / z: >= two launches old
  static constexpr bool kColSums = true;
  __device__ bool want_col_sums() const { return ks == 1; }
  static constexpr bool kMmaReadsRaw = !RES;
  static constexpr int kBox = 32 * kBM * 4;                    // 16 KB
  static constexpr int kBBytes = tc::Tile<BN>::kBytes;
  static constexpr int kRawBytes = 2 * kBox + (RES ? 0 : 2 * kBBytes);
  static constexpr int kNR = IP_ ? 3 : RES ? 3 : (BN <= 64 ? 3 : 2);
  static constexpr int kABytes = tc::Tile<kBM>::kBytes;         // 16 KB
  static constexpr int kOpBytes = 2 * kABytes;
  static constexpr int kNS = IP_ ? 0 : 2;
  static_assert(!IP_ || (!RES && 2 * kBox == kOpBytes), "in place: streamed W1, boxes = operand");
  static constexpr int kNE = 0, kEpiBytes = 0;
  static constexpr bool kEpiStore = false;
  static constexpr int kEpiWarps = 8, kXfWarps = 8;
  static constexpr int kXfThreads = 32 * kXfWarps;
  CUtensorMap xmap;        // feat [M][C] fp32, box {32, 128}, swizzle 128B
  LayerArgs<float> a;
  const uint8_t* w1t;      // pre-tiled W1: per K block, hi tile | lo tile (Tile<BN> K-major)
  // Column split (streamed W1 only): each pixel tile's BN output columns are
  // cut into ns tiles of nw columns, so a block with few pixel tiles (7x7 at
  // batch 64: 25) still spreads over the SMs.  tile = pixel tile * ns + column
  // tile: the ns CTAs of one pixel tile run side by side and share its feature
  // boxes through L2; each streams only its nw columns of W1.  bimg: the
  // column count of the pre-tiled W1 image (>= BN when the template's BN only
  // bounds the column tile, so the streamed stages fit shared memory).
  int ns = 1, nw = BN, bimg = BN;
  // Split-K (streamed W1 only): a pixel tile's K blocks are cut into ks runs
  // of kper blocks, one tile each, so blocks with few pixel tiles (14x14 and
  // 7x7 at batch 64: 98 and 25) spread over the SMs without re-reading the
  // features (the column split re-reads them per column tile).  Each run
  // writes its fp32 partial accumulator to zpart[split][M][bk];
  // k_zsplit_reduce sums them in split order into z and the BN_b partials.
  int ks = 1, kper = 0;
  float* zpart = nullptr;

  __device__ int mtile(int tile) const { return tile / (ns * ks); }
  __device__ int ncol0(int tile) const { return ((tile / ks) % ns) * nw; }
  __device__ int ksplit(int tile) const { return tile % ks; }
  __device__ int kb0(int tile) const { return ks > 1 ? ksplit(tile) * kper : 0; }
  __device__ void prefetch() const { prefetch_tmap(&xmap); }
  __device__ int num_tiles() const { return static_cast<int>((a.M + kBM - 1) / kBM) * ns * ks; }
  __device__ int num_kb(int tile) const {
    const int nkb = (a.c + kBK - 1) / kBK;
    return ks > 1 ? min(kper, nkb - kb0(tile)) : nkb;
  }
  __device__ int boxes(int kb) const { return a.c - kb * kBK > 32 ? 2 : 1; }
  __device__ int epi_chunks(int) const { return nw / 8; }
  __device__ int epi_boxes(int) const { return 0; }
  __device__ void epi_tma(int, int, uint32_t, uint64_t*) const {}
  __device__ void epi_store(int, int, uint32_t) const {}
  __device__ uint32_t raw_bytes(int tile, int kb) const {
    return boxes(kb0(tile) + kb) * kBox + (RES ? 0 : 2 * nw * kBK * 2);
  }
  __device__ uint32_t b_all() const { return static_cast<uint32_t>(((a.c + kBK - 1) / kBK) * 2 * kBBytes); }
  __device__ const BnAff* bn_table(const uint8_t* aux) const {
    return reinterpret_cast<const BnAff*>(aux + (RES ? b_all() : 0));
  }
  __device__ void prologue_early(uint8_t* aux) const {
    if (RES) {
      const uint4* src = reinterpret_cast<const uint4*>(w1t);
      uint4* dst = reinterpret_cast<uint4*>(aux);
      for (int q = threadIdx.x; q < static_cast<int>(b_all() / 16); q += blockDim.x) dst[q] = __ldg(src + q);
    }
  }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_aff(const_cast<BnAff*>(bn_table(aux)), a.c, 0, a.amean, a.avar, a.gamma_a, a.beta_a);
  }
  __device__ void tma(int tile, int kb, uint32_t raw, uint64_t* bar) const {
    const int m0 = mtile(tile) * kBM;
    kb += kb0(tile);  // global K block
    tma_load_2d(raw, &xmap, kb * kBK, m0, bar);
    if (boxes(kb) == 2) tma_load_2d(raw + kBox, &xmap, kb * kBK + 32, m0, bar);
    if (!RES) {
      const uint8_t* src = w1t + static_cast<int64_t>(kb) * 2 * (bimg * kBK * 2);
      if (ns == 1 && bimg == BN) {
        bulk_load(raw + 2 * kBox, src, 2 * kBBytes, bar);
      } else {
        // rows [n0, n0 + nw) of each of the 8 K chunks of the hi and lo tiles:
        // one contiguous nw * 16-byte run each (canonical K-major layout)
        const int n0 = ncol0(tile);
        const uint32_t run = static_cast<uint32_t>(nw) * 16;
#pragma unroll 1
        for (int q = 0; q < 2 * (kBK / 8); ++q)
          bulk_load(raw + 2 * kBox + q * run, src + q * (bimg * 16) + n0 * 16, run, bar);
      }
    }
  }
  __device__ void transform(int tile, int kb, const uint8_t* raw, uint8_t* op, const uint8_t* aux,
                            int xt) const {
    const BnAff* bn = bn_table(aux);
    uint8_t* ah = op;
    uint8_t* al = op + kABytes;
    kb += kb0(tile);  // global K block
    // every chunk of this thread covers the same 8 channels (kmajor_coords):
    // BN as one FMA per element with per-stage register coefficients
    int row0, kc;
    tc::kmajor_coords(xt, row0, kc);
    const int ch0 = kb * kBK + kc;
    float sc[8], sh[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (ch0 + i < a.c) {
        sc[i] = bn[ch0 + i].scale;
        sh[i] = bn[ch0 + i].shift;
      } else {
        sc[i] = 0.f;  // channels past c contribute zero
        sh[i] = 0.f;
      }
    }
    constexpr int kChunks = kBM * kBK / 8 / kXfThreads;
    if constexpr (IP_) {
      // every transform thread reads all of its chunks, the transform warps
      // meet, then the operand overwrites the boxes
      float v[kChunks][8];
#pragma unroll
      for (int i = 0; i < kChunks; ++i) {
        const int row = row0 + i * (kXfThreads / 8);
        if (ch0 < a.c) {
          raw_read8(raw + (kc >> 5) * kBox, row, kc & 31, v[i]);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[i][e] = fmaxf(fmaf(v[i][e], sc[e], sh[e]), 0.f);
        } else {
          tc::zero8(v[i]);
        }
      }
      named_sync(2, kXfThreads);
#pragma unroll
      for (int i = 0; i < kChunks; ++i) {
        const int row = row0 + i * (kXfThreads / 8);
        uint4 h, l;
        tc::split8_h(v[i], h, l);  // fp16x3 forward operands (dpb_tc.cuh)
        const uint32_t off = tc::Tile<kBM>::kmajor_chunk(row, kc);
        tc::st_shared16(ah, off, h);
        tc::st_shared16(al, off, l);
      }
    } else {
#pragma unroll
    for (int i = 0; i < kChunks; ++i) {
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
      tc::split8_h(v, h, l);  // fp16x3 forward operands (dpb_tc.cuh)
      const uint32_t off = tc::Tile<kBM>::kmajor_chunk(row, kc);
      tc::st_shared16(ah, off, h);
      tc::st_shared16(al, off, l);
    }
    }
  }
  __device__ void mma(uint32_t op, uint32_t raw, uint32_t aux, uint32_t tmem, int kb) const {
    const uint32_t ah = op, al = op + kABytes;
    if (RES || (ns == 1 && bimg == BN)) {
      constexpr uint32_t idesc = tc::make_idesc(BN, 0, 0, true);
      const uint32_t bh = RES ? aux + kb * 2 * kBBytes : raw + 2 * kBox, bl = bh + kBBytes;
#pragma unroll
      for (int k16 = 0; k16 < kBK / 16; ++k16) {
        const uint32_t acc = (kb | k16) ? 1u : 0u;
        tc::mma_bf16(tmem, tc::Tile<kBM>::desc(ah, k16), tc::Tile<BN>::desc(bh, k16), idesc, acc);
        tc::mma_bf16(tmem, tc::Tile<kBM>::desc(ah, k16), tc::Tile<BN>::desc(bl, k16), idesc, 1u);
        tc::mma_bf16(tmem, tc::Tile<kBM>::desc(al, k16), tc::Tile<BN>::desc(bh, k16), idesc, 1u);
      }
    } else {
      // streamed column tile: a canonical K-major tile of nw rows
      const uint32_t idesc = tc::make_idesc(nw, 0, 0, true);
      const uint32_t tb = static_cast<uint32_t>(nw) * kBK * 2;
      const uint32_t bh = raw + 2 * kBox, bl = bh + tb;
      const uint32_t k16_step = 2 * static_cast<uint32_t>(nw) * 16, lbo = static_cast<uint32_t>(nw) * 16;
#pragma unroll
      for (int k16 = 0; k16 < kBK / 16; ++k16) {
        const uint32_t acc = (kb | k16) ? 1u : 0u;
        const uint64_t dh = tc::make_sdesc(bh + k16 * k16_step, lbo, 128);
        const uint64_t dl = tc::make_sdesc(bl + k16 * k16_step, lbo, 128);
        tc::mma_bf16(tmem, tc::Tile<kBM>::desc(ah, k16), dh, idesc, acc);
        tc::mma_bf16(tmem, tc::Tile<kBM>::desc(ah, k16), dl, idesc, 1u);
        tc::mma_bf16(tmem, tc::Tile<kBM>::desc(al, k16), dh, idesc, 1u);
      }
    }
  }
  __device__ void epilogue(int tile, int row, int col0, const float (&v)[8], const uint8_t*,
                           uint8_t*, float (&s1)[8], float (&s2)[8]) const {
    const int64_t p = static_cast<int64_t>(mtile(tile)) * kBM + row;
    const int gc = ncol0(tile) + col0;
    const int nv = p < a.M ? min(a.bk - gc, nw - col0) : 0;
    const bool part = ks > 1;  // split-K: the partial accumulator; z and its sums come from the reduce
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = i < nv && !part;
      s1[i] = ok ? v[i] : 0.f;
      s2[i] = ok ? v[i] * v[i] : 0.f;
    }
    if (nv > 0) {
      float* dst = part ? zpart + (static_cast<int64_t>(ksplit(tile)) * a.M + p) * a.bk + gc : a.z + p * a.bk + gc;
      tc::store8(dst, nv, (a.bk & 3) == 0, v);
    }
  }
  __device__ void col_sums(int tile, int c, double s1, double s2) const {
    const int gc = ncol0(tile) + c;
    if (ks == 1 && c < nw && gc < a.bk)
      a.part[static_cast<int64_t>(mtile(tile)) * a.bk + gc] = make_double2(s1, s2);
  }
};

// Split-K 1x1 forward, second pass: z[m][c] = sum over splits of zpart[s][m][c]
// in split order, and the BN_b partial sums (sum z, sum z^2, fp64, fixed
// order) of every kZRows-row block, part[block][c] (the finalize folds
// ceil(M / kZRows) rows).  CTA = kZRows rows x 32 channels (grid.y); 256
// threads = 32 channel lanes x 8 row groups; many small CTAs keep the
// partials' loads in flight (the pass is latency bound).
constexpr int kMaxKSplit = 8, kZRows = 32;
__global__ void __launch_bounds__(256) k_zsplit_reduce(const float* __restrict__ zpart, int ks, int64_t M, int bk,
                                                       float* __restrict__ z, double2* __restrict__ part) {
  pdl_enter();
  __shared__ double r1[8][33], r2[8][33];
  const int lane = threadIdx.x % 32, grp = threadIdx.x / 32;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kZRows;
  const int c = blockIdx.y * 32 + lane;
  double s1 = 0.0, s2 = 0.0;
  if (c < bk) {
    float v[kZRows / 8];
#pragma unroll
    for (int i = 0; i < kZRows / 8; ++i) {
      const int64_t m = m0 + grp + 8 * i;
      float acc = 0.f;
#pragma unroll
      for (int sp = 0; sp < kMaxKSplit; ++sp)
        if (sp < ks && m < M) acc += zpart[(static_cast<int64_t>(sp) * M + m) * bk + c];
      v[i] = acc;
    }
#pragma unroll
    for (int i = 0; i < kZRows / 8; ++i) {
      const int64_t m = m0 + grp + 8 * i;
      if (m < M) {
        z[m * bk + c] = v[i];
        s1 += v[i];
        s2 += static_cast<double>(v[i]) * v[i];
      }
    }
  }
  r1[grp][lane] = s1;
  r2[grp][lane] = s2;
  __syncthreads();
  if (grp == 0 && c < bk) {
    double x = 0.0, y = 0.0;
    for (int g = 0; g < 8; ++g) {
      x += r1[g][lane];
      y += r2[g][lane];
    }
    part[static_cast<int64_t>(blockIdx.x) * bk + c] = make_double2(x, y);
  }
}

// ---- 1x1 backward data: g1 = relu'(act_a) * (t1 . W1) --------------------------------
// N (the layer's c input channels) is split into nn balanced column tiles of nw
// <= BN columns (blockIdx.y = column tile; nw a multiple of 32).
__host__ __device__ inline void bwd_ntiles(int c, int bn_max, int& nn, int& nw) {
  nn = (c + bn_max - 1) / bn_max;
  const int per = (c + nn - 1) / nn;
  nw = (per + 31) / 32 * 32;  // whole 32-column boxes: tile edges are box edges
}
__host__ __device__ inline int bwd_nkb(int bk) { return (bk + 31) / 32; }

// Per pixel tile (128 rows): raw stage = g0 and z boxes of 32 bottleneck
// channels (TMA); the transform warps form t1 = BN_b backward(g0; z) in bf16
// (K-major, K = 32 per stage); the MMA multiplies by the resident pre-tiled
// W1^T column tile (K-major, N = nw).  The epilogue ring streams the layer's
// input features (32-channel boxes of the tile) for the ReLU mask by act_a;
// the epilogue rewrites each feature box in place with g1 (TMA-stored by the
// load warp: whole 128-byte lines, clipped at M and c) and writes the BN_a
// backward column sums (sum g, sum g*xhat) to the tile's partial slot.
// graph.hpp:920-932 / ops.hpp:268-287, 206-243.
// NE_: depth of the feature-box epilogue ring (5: one box of look-ahead over
// the four epilogue groups; 4 frees 16 KB for bk = 192's resident W1^T).
template <int BN_, int NE_ = 5>
struct Dgrad1x1 {
  static constexpr bool kInPlace = false;
  static constexpr int BN = BN_;
  static constexpr int kTmemCols = BN;
  static constexpr bool kEarlyLoads = true;  // g0 (3x3 dgrad) and z: >= two launches old
  static constexpr bool kColSums = true;
  __device__ bool want_col_sums() const { return true; }
  static constexpr bool kMmaReadsRaw = false;
  static constexpr int kBox = 32 * kBM * 4;        // 16 KB: 128 rows x 32 fp32 channels
  static constexpr int kRawBytes = 2 * kBox;       // g0 | z
  static constexpr int kNR = 2;
  static constexpr int kOpBytes = kBM * 32 * 2;    // t1, bf16, 32 K
  static constexpr int kNS = 3;
  static constexpr int kNE = NE_, kEpiBytes = kBox;  // feature boxes, rewritten with g1
  static constexpr bool kEpiStore = true;
  static constexpr int kEpiWarps = 16, kXfWarps = 4;
  static constexpr int kXfThreads = 32 * kXfWarps;
  static constexpr int kBTile = BN * 32 * 2;       // W1^T per 32-K block
  CUtensorMap gmap;   // g0 [M][bk]
  CUtensorMap zmap;   // z_l [M][bk]
  CUtensorMap fmap;   // feat [M][C]
  CUtensorMap omap;   // g1 [M][c]
  LayerArgs<float> a;
  const uint8_t* w1t; // this layer's W1^T tiles: [column tile][kb] Tile<BN> (32 K)
  int nw;             // columns per column tile

  __device__ int n0() const { return blockIdx.y * nw; }
  __device__ int ncols() const { return a.c - n0() < nw ? a.c - n0() : nw; }
  __device__ int nkb() const { return bwd_nkb(a.bk); }
  __device__ void prefetch() const {
    prefetch_tmap(&gmap);
    prefetch_tmap(&zmap);
    prefetch_tmap(&fmap);
    prefetch_tmap(&omap);
  }
  __device__ int num_tiles() const { return static_cast<int>((a.M + kBM - 1) / kBM); }
  __device__ int num_kb(int) const { return nkb(); }
  __device__ uint32_t raw_bytes(int, int) const { return 2 * kBox; }
  __device__ int epi_chunks(int) const { return (ncols() + 7) / 8; }
  __device__ int epi_boxes(int) const { return (ncols() + 31) / 32; }
  __device__ const BnBwd* bnb(const uint8_t* aux) const {
    return reinterpret_cast<const BnBwd*>(aux + nkb() * kBTile);
  }
  __device__ const float4* bna(const uint8_t* aux) const {  // mask form (fill_bn_mask4)
    return reinterpret_cast<const float4*>(aux + nkb() * kBTile + ((sizeof(BnBwd) * a.bk + 15) / 16) * 16);
  }
  __device__ void prologue_early(uint8_t* aux) const {
    const uint4* src = reinterpret_cast<const uint4*>(w1t + static_cast<int64_t>(blockIdx.y) * nkb() * kBTile);
    uint4* dst = reinterpret_cast<uint4*>(aux);
    for (int q = threadIdx.x; q < nkb() * kBTile / 16; q += blockDim.x) dst[q] = __ldg(src + q);
    // BN_a forward statistics and parameters: old
    fill_bn_mask4(const_cast<float4*>(bna(aux)), ncols(), n0(), a.amean, a.avar, a.gamma_a, a.beta_a);
  }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_bwd(const_cast<BnBwd*>(bnb(aux)), a);  // the BN_b coefficients: the predecessor's output
  }
  __device__ void tma(int tile, int kb, uint32_t raw, uint64_t* bar) const {
    tma_load_2d(raw, &gmap, kb * 32, tile * kBM, bar);
    tma_load_2d(raw + kBox, &zmap, kb * 32, tile * kBM, bar);
  }
  __device__ void epi_tma(int tile, int b, uint32_t dst, uint64_t* bar) const {
    tma_load_2d(dst, &fmap, n0() + b * 32, tile * kBM, bar);
  }
  __device__ void epi_store(int tile, int b, uint32_t src) const {
    tc::tma_store_2d(&omap, src, n0() + b * 32, tile * kBM);
  }
  __device__ void transform(int, int kb, const uint8_t* raw, uint8_t* op, const uint8_t* aux,
                            int xt) const {
    const BnBwd* bb = bnb(aux);
#pragma unroll
    for (int i = 0; i < kBM * 32 / 8 / kXfThreads; ++i) {
      // a phase of 8 threads writes one whole core matrix (conflict free)
      const int q = xt + i * kXfThreads;
      const int row = (q & 7) | (((q >> 3) & 15) << 3);
      const int kc = ((q >> 7) & 3) << 3;
      const int j0 = kb * 32 + kc;
      float v[8];
      if (j0 < a.bk) {
        float zz[8];
        raw_read8(raw, row, kc, v);
        raw_read8(raw + kBox, row, kc, zz);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = j0 + e < a.bk ? bnb_t1(bb[j0 + e], v[e], zz[e]) : 0.f;
      } else {
        tc::zero8(v);
      }
      tc::st_shared16(op, tc::Tile<kBM>::kmajor_chunk(row, kc), tc::to_bf16x8(v));
    }
  }
  __device__ void mma(uint32_t op, uint32_t, uint32_t aux, uint32_t tmem, int kb) const {
    const uint32_t idesc = tc::make_idesc(nw, 0, 0);
    const uint32_t b = aux + kb * kBTile;
#pragma unroll
    for (int k16 = 0; k16 < 2; ++k16)
      if (kb * 32 + k16 * 16 < a.bk)
        tc::mma_bf16(tmem, tc::Tile<kBM>::desc(op, k16), tc::Tile<BN>::desc(b, k16), idesc,
                     (kb | k16) ? 1u : 0u);
  }
  __device__ void epilogue(int tile, int row, int col0, const float (&v)[8], const uint8_t* aux,
                           uint8_t* ebox, float (&s1)[8], float (&s2)[8]) const {
    const float4* bn = bna(aux);
    const int64_t p = static_cast<int64_t>(tile) * kBM + row;
    const int rem = ncols() - col0;
    const int nv = p < a.M ? (rem < 8 ? rem : 8) : 0;
    float x[8], g[8];
    raw_read8(ebox, row, col0 & 31, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < nv) {
        const float4 b = bn[col0 + i];
        g[i] = relu_mask4(b, x[i]) ? v[i] : 0.f;  // relu_backward by act_a
        s1[i] = g[i];
        s2[i] = g[i] * ((x[i] - b.x) * b.y);
      } else {
        g[i] = 0.f;
        s1[i] = 0.f;
        s2[i] = 0.f;
      }
    }
    // g over x in the staging box; columns past nv are outside [0, M) x [0, c)
    // here (tile edges are box edges) and are clipped by the store
    raw_write8(ebox, row, col0 & 31, g);
  }
  __device__ void col_sums(int tile, int c, double s1, double s2) const {
    if (c < ncols()) a.part[static_cast<int64_t>(tile) * a.c + n0() + c] = make_double2(s1, s2);
  }
};

// ---- 1x1 backward weights: dW1[j][i] = sum_p t1[p,j] act_a[p,i] ------------------------
// Split-K over pixels: CTA x owns pixel blocks [x*kchunk, ...) of 32 pixels
// (ONE engine tile per CTA, so the accumulator stays in TMEM across the whole
// range), blockIdx.y the column tile of input channels.  Per block the raw
// stage holds 32-pixel TMA boxes of g0 and z (JB boxes of 32 bottleneck
// channels each) and of the features (BN/32 boxes); the transform warps form
// t1^T (A: M = j, K = p, MN-major) and act_a = relu(bn_a(x)) (B: N = i, K = p,
// MN-major) in bf16.  M = j runs over kMT tiles of 128.  The epilogue writes
// the CTA's partial dW1 [split][j][i] (rows j < bk, columns i < the tile's
// width); k_reduce_w1 folds the splits.  graph.hpp:920-922, ops.hpp:330-387.
template <int BN_, int JB>
struct Wgrad1x1 {
  static constexpr bool kInPlace = false;
  static constexpr int BN = BN_;
  static constexpr int kMT = (JB * 32 + 127) / 128;
  static constexpr int kTmemCols = kMT * BN;
  static constexpr bool kEarlyLoads = false;  // side stream: behind an event, not a PDL edge
  static constexpr bool kColSums = false;
  __device__ bool want_col_sums() const { return false; }
  static constexpr bool kMmaReadsRaw = false;
  static constexpr int kBoxP = 32;                       // pixels per K block
  static constexpr int kBox = kBoxP * 32 * 4;            // 4 KB
  static constexpr int kRawBytes = (2 * JB + BN / 32) * kBox;
  static constexpr int kNR = kRawBytes <= 48 * 1024 ? 3 : 2;
  static constexpr int kATile = kBM * kBoxP * 2;         // 8 KB per M tile
  static constexpr int kOpBytes = kMT * kATile + BN * kBoxP * 2;
  static constexpr int kNS = 2;
  static constexpr int kNE = 0, kEpiBytes = 0;
  static constexpr bool kEpiStore = false;
  static constexpr int kEpiWarps = 4, kXfWarps = 8;
  static constexpr int kXfThreads = 32 * kXfWarps;
  CUtensorMap gmap, zmap, fmap;  // g0, z_l [M][bk]; feat [M][C]; box {32, 32}
  LayerArgs<float> a;
  int nw;       // columns per column tile
  int kchunk;   // pixel blocks per CTA
  int nblk;     // pixel blocks in total

  __device__ int n0() const { return blockIdx.y * nw; }
  __device__ int ncols() const { return a.c - n0() < nw ? a.c - n0() : nw; }
  __device__ int jboxes() const { return (a.bk + 31) / 32; }
  __device__ int fboxes() const { return (ncols() + 31) / 32; }
  __device__ void prefetch() const {
    prefetch_tmap(&gmap);
    prefetch_tmap(&zmap);
    prefetch_tmap(&fmap);
  }
  __device__ int num_tiles() const { return gridDim.x; }
  __device__ int num_kb(int tile) const {
    const int rest = nblk - tile * kchunk;
    return rest < kchunk ? rest : kchunk;
  }
  __device__ uint32_t raw_bytes(int, int) const { return (2 * jboxes() + fboxes()) * kBox; }
  __device__ int epi_chunks(int) const { return kMT * BN / 8; }
  __device__ int epi_boxes(int) const { return 0; }
  __device__ void epi_tma(int, int, uint32_t, uint64_t*) const {}
  __device__ void epi_store(int, int, uint32_t) const {}
  __device__ const BnBwd* bnb(const uint8_t* aux) const { return reinterpret_cast<const BnBwd*>(aux); }
  __device__ const float4* bna(const uint8_t* aux) const {  // apply form (fill_bn_apply4)
    return reinterpret_cast<const float4*>(aux + ((sizeof(BnBwd) * a.bk + 15) / 16) * 16);
  }
  __device__ void prologue_early(uint8_t*) const {}
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_bwd(const_cast<BnBwd*>(bnb(aux)), a);
    fill_bn_apply4(const_cast<float4*>(bna(aux)), ncols(), n0(), a.amean, a.avar, a.gamma_a, a.beta_a);
  }
  __device__ void tma(int tile, int kb, uint32_t raw, uint64_t* bar) const {
    const int p0 = (tile * kchunk + kb) * kBoxP;
    for (int jb = 0; jb < jboxes(); ++jb) {
      tma_load_2d(raw + jb * kBox, &gmap, jb * 32, p0, bar);
      tma_load_2d(raw + (JB + jb) * kBox, &zmap, jb * 32, p0, bar);
    }
    for (int fb = 0; fb < fboxes(); ++fb) tma_load_2d(raw + (2 * JB + fb) * kBox, &fmap, n0() + fb * 32, p0, bar);
  }
  __device__ void transform(int tile, int kb, const uint8_t* raw, uint8_t* op, const uint8_t* aux,
                            int xt) const {
    const int64_t p0 = static_cast<int64_t>(tile * kchunk + kb) * kBoxP;
    const int jc = (a.bk + 7) / 8, ic = (ncols() + 7) / 8;
    const BnBwd* bb = bnb(aux);
    const float4* bn = bna(aux);
    // 8 consecutive chunks = 8 consecutive pixels of one channel group: one
    // whole MN-major core matrix per store phase, conflict-free box reads
    for (int q = xt; q < kBoxP * (jc + ic); q += kXfThreads) {
      const int p = q & (kBoxP - 1);
      const int grp = q / kBoxP;
      float v[8];
      if (grp < jc) {
        const int j0 = grp * 8;
        float zz[8];
        raw_read8(raw + (j0 >> 5) * kBox, p, j0 & 31, v);
        raw_read8(raw + (JB + (j0 >> 5)) * kBox, p, j0 & 31, zz);
        const bool live = p0 + p < a.M;
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = live && j0 + e < a.bk ? bnb_t1(bb[j0 + e], v[e], zz[e]) : 0.f;
        tc::st_shared16(op + (j0 >> 7) * kATile, tc::Tile<kBM>::mnmajor_chunk(j0 & 127, p), tc::to_bf16x8(v));
      } else {
        const int i0 = (grp - jc) * 8;
        raw_read8(raw + (2 * JB + (i0 >> 5)) * kBox, p, i0 & 31, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 b = bn[i0 + e < ncols() ? i0 + e : 0];
          v[e] = fmaxf(fmaf(v[e] - b.x, b.y, b.z), 0.f);  // act_a (t1 is 0 past M)
        }
        tc::st_shared16(op + kMT * kATile, tc::Tile<BN>::mnmajor_chunk(i0, p), tc::to_bf16x8(v));
      }
    }
  }
  __device__ void mma(uint32_t op, uint32_t, uint32_t, uint32_t tmem, int kb) const {
    const uint32_t idesc = tc::make_idesc(nw, 1, 1);
    const uint32_t b = op + kMT * kATile;
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
      for (int k16 = 0; k16 < kBoxP / 16; ++k16)
        tc::mma_bf16(tmem + mt * BN, tc::Tile<kBM>::desc(op + mt * kATile, k16), tc::Tile<BN>::desc(b, k16),
                     idesc, (kb | k16) ? 1u : 0u);
  }
  __device__ void epilogue(int tile, int row, int col0, const float (&v)[8], const uint8_t*, uint8_t*,
                           float (&)[8], float (&)[8]) const {
    const int mt = col0 / BN;
    const int i0 = col0 - mt * BN;
    const int j = mt * kBM + row;
    if (j < a.bk && i0 < ncols()) {
      const int nv = ncols() - i0 < 8 ? ncols() - i0 : 8;
      tc::store8(a.wpart + (static_cast<int64_t>(tile) * a.bk + j) * a.c + n0() + i0, nv, (a.c & 3) == 0, v);
    }
  }
  __device__ void col_sums(int, int, double, double) const {}
};

// W1^T operand images of every layer for Dgrad1x1<BN> (blockIdx.y = layer):
// per column tile and 32-K block, Tile<BN> K-major with rows = input channels
// i, K = bottleneck channels j; zero outside [0, c) x [0, bk).
template <int BN>
__global__ void k_pretile_w1t_all(const float* __restrict__ params, int c0, int k, int bk,
                                  uint8_t* __restrict__ out) {
  pdl_enter();
  const int l = blockIdx.y;
  const int nkb = bwd_nkb(bk);
  int64_t poff = 0, toff = 0;
  for (int j = 0; j < l; ++j) {
    const int cj = c0 + j * k;
    int nn, nw;
    bwd_ntiles(cj, BN, nn, nw);
    poff += 2LL * cj + static_cast<int64_t>(bk) * cj + 2LL * bk + 9LL * k * bk;
    toff += static_cast<int64_t>(nn) * nkb * BN * 64;
  }
  const int c = c0 + l * k;
  int nn, nw;
  bwd_ntiles(c, BN, nn, nw);
  const float* w1 = params + poff + 2 * c;
  const int chunks = BN * 4;  // 8-element chunks per (tile, kb)
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nn * nkb * chunks; q += gridDim.x * blockDim.x) {
    const int t = q / chunks, qq = q - t * chunks;
    const int nt = t / nkb, kb = t - nt * nkb;
    const int n = qq >> 2, kc = (qq & 3) << 3;
    const int i = nt * nw + n;
    const int j0 = kb * 32 + kc;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      v[e] = (n < nw && i < c && j0 + e < bk) ? w1[static_cast<int64_t>(j0 + e) * c + i] : 0.f;
    *reinterpret_cast<uint4*>(out + toff + static_cast<int64_t>(t) * BN * 64 +
                              tc::Tile<BN>::kmajor_chunk(n, kc)) = tc::to_bf16x8(v);
  }
}

// All layers of a block in one launch: blockIdx.y = layer.
template <int BN>
__global__ void k_pretile_w1_all(const float* __restrict__ params, int c0, int k, int bk, int m,
                                 uint8_t* __restrict__ out) {
  pdl_enter();
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
    tc::split8_h(v, h, lo);  // W1 hi | lo, fp16 (the forward's fp16x3)
    uint8_t* t = out + toff + static_cast<int64_t>(kb) * 2 * tc::Tile<BN>::kBytes;
    const uint32_t off = tc::Tile<BN>::kmajor_chunk(row, kc);
    *reinterpret_cast<uint4*>(t + off) = h;
    *reinterpret_cast<uint4*>(t + tc::Tile<BN>::kBytes + off) = lo;
  }
}

}  // namespace tc2
}  // namespace dpb
