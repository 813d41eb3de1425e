// 3x3 convolutions as tcgen05 GEMMs over a haloed tile in a PADDED pixel space.
//
// Each image is viewed as (H+2) x (W+2) padded positions with zero borders.  A
// CTA owns 128 consecutive positions of one image's band (padded rows 1..H,
// all W+2 columns).  Its producers transform the tile's halo — positions
// [s0 - (W+3), s0 + 128 + (W+3)) — ONCE into shared memory (BN+ReLU or plain
// bf16, zeros at padding), in a layout whose rows are 16 bytes apart.  A 3x3
// tap (dy, dx) is then a pure row shift: the UMMA descriptor's start address
// moves by (dy*(W+2) + dx) * 16 bytes.  So the 9x re-gather of the shifted
// operand that a plain implicit GEMM pays disappears; zero padding AFTER the
// activation is physical in the halo.  Outputs on padding columns are
// computed and dropped (2/(W+2) of the rows).
//
//   Tc3x3FwdHalo   D[pos][o]        = sum_tap sum_j act_b[pos+d][j] W2[o][j][tap]  (bf16x3)
//   Tc3x3DgradHalo D[pos][j]        = sum_tap sum_o dY[pos-d][o]    W2[o][j][tap]  (bf16)
//   Tc3x3WgradHalo D_tap[j][o]      = sum_pos act_b[pos+d][j] dY[pos][o]          (bf16,
//                                     9 TMEM accumulators, split-K over tiles)
// Reference semantics: /root/reference/proj/include/denseplan/ops.hpp:315-387
// (conv2d_forward / conv2d_backward, padding 1) inside graph.hpp:655, :906-907.
#pragma once

#include "dpb_simt.cuh"
#include "dpb_tc.cuh"

namespace dpb {
namespace tc {

// Geometry of the padded band shared by the three ops.
struct HaloGeom {
  int H, W, W2;     // W2 = W + 2
  int tpi;          // tiles per image = ceil(H * W2 / 128)
  int R;            // halo rows = 128 + 2 * (W2 + 1), rounded up to 8
  __host__ __device__ static HaloGeom make(int H, int W) {
    HaloGeom g;
    g.H = H;
    g.W = W;
    g.W2 = W + 2;
    g.tpi = (H * g.W2 + kBM - 1) / kBM;
    g.R = (kBM + 2 * (g.W2 + 1) + 7) / 8 * 8;
    return g;
  }
  // padded position of halo row r of tile t (may be < 0 or past the image)
  __device__ int pos(int t, int r) const { return g_s0(t) - (W2 + 1) + r; }
  __device__ int g_s0(int t) const { return W2 + t * kBM; }
  // real pixel (within the image) of padded position q, or -1 for padding
  __device__ int pixel(int q) const {
    if (q < 0) return -1;
    const int py = q / W2, px = q - py * W2;
    if (py < 1 || py > H || px < 1 || px > W) return -1;
    return (py - 1) * W + (px - 1);
  }
  // halo-row offset of tap (ty, tx) for the forward (source = pos + d)
  __device__ int fwd_off(int tap) const { return (W2 + 1) + (tap / 3 - 1) * W2 + (tap % 3 - 1); }
  // ... and for the transposed conv (source = pos - d)
  __device__ int bwd_off(int tap) const { return (W2 + 1) - (tap / 3 - 1) * W2 - (tap % 3 - 1); }
};

// K-major halo tile: element (row, k) at (k/8)*R*16 + row*16 + (k%8)*2.
__device__ __forceinline__ uint32_t halo_kmajor(int R, int row, int k) {
  return static_cast<uint32_t>((k >> 3) * R * 16 + row * 16);
}
// MN-major halo tile (rows = channels j, K = positions): element (j, pos) at
// (j/8)*R*16 + pos*16 + (j%8)*2.
__device__ __forceinline__ uint32_t halo_mnmajor(int R, int j, int pos) {
  return static_cast<uint32_t>((j >> 3) * R * 16 + pos * 16);
}

// Debug phase clocks (dpb_debug_phase_clocks): thread 0 of the first 4096
// CTAs records clock64 stamps at the phase boundaries: start, prologue done,
// last produce, last issue, MMAs complete, epilogue loop done, epilogue
// barrier passed, column sums written, exit.
__device__ long long g_phase_clock[4096][9];
__device__ long long g_kb_clock[4096][8][4];  // per K chunk: stage free, produced, barrier, weights landed
__device__ int g_phase_on;

// ---- engine ----------------------------------------------------------------------
// As tc_gemm_kernel, but the op owns the stage layout and the MMA issue
// pattern (taps = descriptor shifts), and TMEM may hold several accumulators.
template <class Op>
__global__ void __launch_bounds__(kThreads, Op::kMinBlocks) tc_halo_kernel(const Op op) {
  constexpr uint32_t TCOLS = TmemCols<Op::kTmemCols>::value;
  constexpr int BN = Op::BN;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint64_t bbar[2];  // async bulk copies of pre-tiled weight images
  __shared__ uint64_t fbar[2];  // kSpecialized: stage's halo produced (one arrive per producer warp)
  __shared__ uint32_t tmem_base;
  __shared__ float red[2][4][BN];

  const int tid = threadIdx.x;
  const int warp = tid / 32, lane = tid % 32;
  // g_phase_on: 1 stamps the ops with column sums (forward, dgrad), 2 the wgrad.
  // Compiled in only with DPB_PHASE_CLOCKS: reading the flag is a global load
  // at kernel entry that every CTA would wait on.
#ifdef DPB_PHASE_CLOCKS
  const bool dbg = g_phase_on == (Op::kColSums ? 1 : 2) && tid == 0 && blockIdx.x + blockIdx.y * gridDim.x < 4096;
#else
  constexpr bool dbg = false;
#endif
  const int dbg_id = blockIdx.x + blockIdx.y * gridDim.x;
  if (dbg) g_phase_clock[dbg_id][0] = clock64();
  const uint32_t SB = op.stage_bytes();
  const int nst = op.num_kb() > 1 ? 2 : 1;  // stages actually used
  uint8_t* aux = smem + nst * SB;

  if (warp == 0) tmem_alloc<TCOLS>(&tmem_base);
  if (tid == 32) {
    // each stage completes when every issuing warp's MMAs have completed
    mbar_init(&mbar[0], Op::kIssuers);
    mbar_init(&mbar[1], Op::kIssuers);
    mbar_init(&bbar[0], 1);
    mbar_init(&bbar[1], 1);
    mbar_init(&fbar[0], 8 - Op::kIssuers);
    mbar_init(&fbar[1], 8 - Op::kIssuers);
    fence_barrier_init();
  }
  // tables built from data two or more launches old (see dpb_tc2.cuh) are
  // filled before the grid-dependency wait
  if constexpr (Op::kEarlyPrologue) op.prologue(aux);
  pdl_enter();  // barrier init / TMEM alloc / early tables above overlap the predecessor
  if constexpr (!Op::kEarlyPrologue) op.prologue(aux);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (dbg) g_phase_clock[dbg_id][1] = clock64();

  const int nkb = op.num_kb();
  if constexpr (Op::kSpecialized) {
    // warps [0, kIssuers) issue, the others produce; stages are handed off by
    // mbarriers (fbar: halo produced, bbar: weights landed, mbar: MMAs done),
    // so the producers build chunk kb+1 while chunk kb's MMAs are issued and
    // run, and weights for kb+1 load as soon as kb-1's MMAs release the stage
    if (warp < Op::kIssuers) {
      if (lane == 0) {
        if (tid == 0) {
          op.bulk(smem_u32(smem), 0, &bbar[0]);
          if (nkb > 1) op.bulk(smem_u32(smem + SB), 1, &bbar[1]);
        }
        for (int kb = 0; kb < nkb; ++kb) {
          const int s = kb & 1;
          mbar_wait(&fbar[s], (kb >> 1) & 1);
          mbar_wait(&bbar[s], (kb >> 1) & 1);
          if (dbg && kb < 8) g_kb_clock[dbg_id][kb][3] = clock64();
          tc_fence_after();
          op.issue(smem_u32(smem + s * SB), kb, tmem, warp);
          mma_commit(&mbar[s]);
          if (tid == 0 && kb >= 1 && kb + 1 < nkb) {  // stage (kb+1)&1 free once kb-1's MMAs completed
            const int s1 = (kb + 1) & 1;
            mbar_wait(&mbar[s1], ((kb - 1) >> 1) & 1);
            op.bulk(smem_u32(smem + s1 * SB), kb + 1, &bbar[s1]);
          }
        }
      }
    } else {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb & 1;
        if (kb >= 2) mbar_wait(&mbar[s], ((kb - 2) >> 1) & 1);
        op.produce(smem + s * SB, kb, aux);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&fbar[s]);
      }
    }
    if (dbg) g_phase_clock[dbg_id][2] = g_phase_clock[dbg_id][3] = clock64();
  }
  for (int kb = 0; !Op::kSpecialized && kb < nkb; ++kb) {
    const int s = kb & 1;
    if (kb >= 2) mbar_wait(&mbar[s], ((kb - 2) >> 1) & 1);
    if (dbg && kb < 8) g_kb_clock[dbg_id][kb][0] = clock64();
    uint8_t* st = smem + s * SB;
    if constexpr (Op::kBulk)
      if (tid == 0) op.bulk(smem_u32(st), kb, &bbar[s]);
    op.produce(st, kb, aux);
    if (dbg && kb < 8) g_kb_clock[dbg_id][kb][1] = clock64();
    fence_proxy_async();
    __syncthreads();
    if (dbg && kb < 8) g_kb_clock[dbg_id][kb][2] = clock64();
    if (dbg && kb == nkb - 1) g_phase_clock[dbg_id][2] = clock64();
    // the MMAs are issued by lane 0 of kIssuers warps in parallel (each into
    // its own accumulator or disjoint columns): a tcgen05.mma issue costs
    // ~60 cycles of uniform-register setup, several times the execution time
    // of these narrow-N MMAs
    if (lane == 0 && warp < Op::kIssuers) {
      if constexpr (Op::kBulk) mbar_wait(&bbar[s], (kb >> 1) & 1);
      if (dbg && kb < 8) g_kb_clock[dbg_id][kb][3] = clock64();
      tc_fence_after();
      op.issue(smem_u32(st), kb, tmem, warp);
      mma_commit(&mbar[s]);
    }
    if (dbg && kb == nkb - 1) g_phase_clock[dbg_id][3] = clock64();
  }
  if (nkb > 0) {
    mbar_wait(&mbar[(nkb - 1) & 1], ((nkb - 1) >> 1) & 1);
    tc_fence_after();
  }
  if (dbg) g_phase_clock[dbg_id][4] = clock64();

  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  // K pair (ops with kKPair, op.kpair set): the two CTAs of a cluster (1, 2)
  // each accumulated half of the K chunks of one tile; rank 1 adds its
  // accumulator into rank 0's shared exchange buffer over DSMEM and leaves,
  // rank 0 runs the epilogue on the sum.  (Fixed order: rank 0 + rank 1.)
  const float* xsum = nullptr;
  if constexpr (Op::kKPair) {
    if (op.kpair) {
      constexpr int kCols = Op::kTmemCols / Op::kAccCopies;
      float* xbuf = reinterpret_cast<float*>(aux + op.xbuf_offset());  // [kBM][kCols]
      const uint32_t rank = cluster_ctarank();
      if (rank == 1) {
        for (int cc = half; cc < kCols / 8; cc += 2) {
          float v[8];
          tmem_ld8(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cc * 8, v);
#pragma unroll
          for (int c2 = 1; c2 < Op::kAccCopies; ++c2) {
            float w[8];
            tmem_ld8(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c2 * kCols + cc * 8, w);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += w[i];
          }
          const uint32_t dst = mapa_cluster(smem_u32(xbuf + row * kCols + cc * 8), 0);
          st_cluster_v4(dst, v[0], v[1], v[2], v[3]);
          st_cluster_v4(dst + 16, v[4], v[5], v[6], v[7]);
        }
      }
      cluster_sync();  // release rank 1's stores / acquire them on rank 0
      if (rank == 1) {
        tc_fence_before();
        __syncthreads();
        if (warp == 0) {
          tc_fence_after();
          tmem_dealloc<TCOLS>(tmem);
        }
        return;
      }
      xsum = xbuf;
    }
  }
  float* ytap = reinterpret_cast<float*>(smem);  // kTapCols: [9][128][k], over the dead stages
  if constexpr (Op::kTapCols) {
    // all taps in one GEMM: D[r][tap*k + o] over halo rows r (M blocks of 128);
    // y[p] = sum_tap D[p + off_tap][tap*k + o].  Each tap's rows land in their
    // own slice (a bijection r -> p, no write conflicts, no barriers between
    // taps); the output pass sums the slices in tap order (deterministic).
    const int mb = warp >> 2;  // M block of this warp (TMEM lanes = its quarter)
    const int r = mb * kBM + row;
    const int k = op.tap_k();
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + mb * kBM;
#pragma unroll 1
    for (int t0 = 0; t0 < 9; t0 += 3) {
      uint32_t u[3][4][4];
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * i < k) tmem_ld4_nowait(lane_base + op.tap_col(t0 + t) + 4 * i, u[t][i]);
      tmem_wait_ld();
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int p = r - op.tap_off(t0 + t);
        if (p >= 0 && p < kBM && r < op.rows()) {
          float* dst = ytap + ((t0 + t) * kBM + p) * k;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (4 * i < k)
              reinterpret_cast<float4*>(dst)[i] =
                  make_float4(__uint_as_float(u[t][i][0]), __uint_as_float(u[t][i][1]),
                              __uint_as_float(u[t][i][2]), __uint_as_float(u[t][i][3]));
        }
      }
    }
    __syncthreads();
  }
  constexpr int kOutCols = Op::kTapCols ? BN : Op::kTmemCols / Op::kAccCopies;  // summed copies
  if constexpr (Op::kEpiPrefetch > 0) {
    // the op's per-row global operand (e.g. the dgrad's z) for kEpiPrefetch
    // column groups is loaded before their TMEM reads: one memory latency per
    // batch instead of one per group
    constexpr int PF = Op::kEpiPrefetch;
    for (int cb = half; cb < kOutCols / 8; cb += 2 * PF) {
      float pre[PF][8];
#pragma unroll
      for (int i = 0; i < PF; ++i)
        if (cb + 2 * i < kOutCols / 8) op.epi_load(row, (cb + 2 * i) * 8, pre[i]);
#pragma unroll
      for (int i = 0; i < PF; ++i) {
        const int cc = cb + 2 * i;
        if (cc >= kOutCols / 8) break;
        float v[8];
        tmem_ld8(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cc * 8, v);
        float s1[8], s2[8];
        op.epilogue_pre(row, cc * 8, v, aux, pre[i], s1, s2);
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
    }
  }
  for (int cc = half; Op::kEpiPrefetch == 0 && cc < kOutCols / 8; cc += 2) {
    float v[8];
    if constexpr (Op::kTapCols) {
      // 16-byte reads (row stride k floats, k % 4 == 0: conflict-free phases)
      const int k = op.tap_k();
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
#pragma unroll
      for (int h4 = 0; h4 < 2; ++h4) {
        if (cc * 8 + 4 * h4 < k) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const float4 q = *reinterpret_cast<const float4*>(ytap + (tap * kBM + row) * k + cc * 8 + 4 * h4);
            v[4 * h4 + 0] += q.x;
            v[4 * h4 + 1] += q.y;
            v[4 * h4 + 2] += q.z;
            v[4 * h4 + 3] += q.w;
          }
        }
      }
    } else if (nkb > 0) {
      tmem_ld8(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cc * 8, v);
#pragma unroll
      for (int c2 = 1; c2 < Op::kAccCopies; ++c2) {
        float w[8];
        tmem_ld8(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c2 * kOutCols + cc * 8, w);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += w[i];
      }
      if (xsum) {  // K pair: + the partner CTA's half
        const float4 a = *reinterpret_cast<const float4*>(xsum + row * kOutCols + cc * 8);
        const float4 b = *reinterpret_cast<const float4*>(xsum + row * kOutCols + cc * 8 + 4);
        v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
        v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
      }
    } else {
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
    }
    float s1[8], s2[8];
    op.epilogue(row, cc * 8, v, aux, s1, s2);
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
  if (dbg) g_phase_clock[dbg_id][5] = clock64();
  tc_fence_before();
  __syncthreads();
  if (dbg) g_phase_clock[dbg_id][6] = clock64();
  if constexpr (Op::kColSums) {
    for (int c = tid; c < BN; c += kThreads) {
      const double a = static_cast<double>(red[0][0][c]) + red[0][1][c] + red[0][2][c] + red[0][3][c];
      const double b = static_cast<double>(red[1][0][c]) + red[1][1][c] + red[1][2][c] + red[1][3][c];
      op.col_sums(c, a, b);
    }
  }
  if (dbg) g_phase_clock[dbg_id][7] = clock64();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<TCOLS>(tmem);
  }
  if (dbg) g_phase_clock[dbg_id][8] = clock64();
}

struct HaloArgs {
  LayerArgs<float> a;
  HaloGeom g;
  int kc;    // channels per K chunk (forward) / padded k (backward), multiple of 16
  int vec;   // 16-byte aligned feature / accumulator rows at channel c
  const uint8_t* wt;  // pre-tiled W2 operand image of this layer (smem layout)
};

// Copy `bytes` (multiple of 16) of a pre-tiled operand image into shared memory.
__device__ __forceinline__ void copy_image(uint8_t* dst, const uint8_t* src, int bytes) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (int q = threadIdx.x; q < bytes / 16; q += kThreads) d[q] = __ldg(s + q);
}

// W2 for the halo forward: per K chunk kb of kc channels, rows tap*BN + o,
// K-major (R = 9*BN), bf16 hi plane then lo plane.
template <int BN>
__global__ void k_pretile_w2_fwd(const float* __restrict__ params, int c0, int k, int bk, int kc,
                                 uint8_t* __restrict__ out) {
  pdl_enter();
  const int l = blockIdx.y;
  int64_t poff = 0;
  for (int j = 0; j < l; ++j) {
    const int cj = c0 + j * k;
    poff += 2LL * cj + static_cast<int64_t>(bk) * cj + 2LL * bk + 9LL * k * bk;
  }
  const int c = c0 + l * k;
  const float* w2 = params + poff + 2 * c + static_cast<int64_t>(bk) * c + 2 * bk;
  const int nkb = (bk + kc - 1) / kc;
  const int plane = 9 * BN * kc * 2;
  uint8_t* o_l = out + static_cast<int64_t>(l) * nkb * 2 * plane;
  const int kcn = kc / 8;
  const int per = 9 * BN * kcn;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nkb * per; q += gridDim.x * blockDim.x) {
    const int kb = q / per, qq = q - kb * per;
    const int row = qq / kcn, kk = (qq % kcn) * 8;
    const int tap = row / BN, o = row - tap * BN;
    const int j0 = kb * kc + kk;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = (o < k && j0 + i < bk) ? w2[(static_cast<int64_t>(o) * bk + j0 + i) * 9 + tap] : 0.f;
    uint4 h, lo;
    split8_h(v, h, lo);  // fp16x3 forward operands (dpb_tc.cuh)
    uint8_t* t = o_l + static_cast<int64_t>(kb) * 2 * plane;
    const uint32_t off = halo_kmajor(9 * BN, row, kk);
    *reinterpret_cast<uint4*>(t + off) = h;
    *reinterpret_cast<uint4*>(t + plane + off) = lo;
  }
}

// W2^T for the halo dgrad: rows tap*BN + j, K = o (kc = k padded), bf16.
template <int BN>
__global__ void k_pretile_w2_bwd(const float* __restrict__ params, int c0, int k, int bk, int kc, int nh,
                                 uint8_t* __restrict__ out) {
  pdl_enter();
  const int l = blockIdx.y;
  int64_t poff = 0;
  for (int j = 0; j < l; ++j) {
    const int cj = c0 + j * k;
    poff += 2LL * cj + static_cast<int64_t>(bk) * cj + 2LL * bk + 9LL * k * bk;
  }
  const int c = c0 + l * k;
  const float* w2 = params + poff + 2 * c + static_cast<int64_t>(bk) * c + 2 * bk;
  // nh column groups of BN (the dgrad's grid.y), each its own contiguous image
  uint8_t* o_l = out + static_cast<int64_t>(l) * nh * 9 * BN * kc * 2;
  const int kcn = kc / 8;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nh * 9 * BN * kcn; q += gridDim.x * blockDim.x) {
    const int hg = q / (9 * BN * kcn), qr = q - hg * (9 * BN * kcn);
    const int row = qr / kcn, kk = (qr % kcn) * 8;
    const int tap = row / BN, j = hg * BN + row - tap * BN;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = (j < bk && kk + i < k) ? w2[(static_cast<int64_t>(kk + i) * bk + j) * 9 + tap] : 0.f;
    *reinterpret_cast<uint4*>(o_l + static_cast<int64_t>(hg) * 9 * BN * kc * 2 + halo_kmajor(9 * BN, row, kk)) =
        to_bf16x8(v);
  }
}

// ---- forward ------------------------------------------------------------------------
// y = conv3x3(relu(bn_b(z))): per K chunk of kc channels the stage holds the
// halo (hi, lo) and W2 for all 9 taps (hi, lo).  The W2 image arrives by an
// asynchronous bulk copy while the threads build the halo; each thread issues
// all of its halo loads before converting any (one memory latency per stage).
#ifndef DPB_FWD_ISSUERS
#define DPB_FWD_ISSUERS 2
#endif
template <int BN_>
struct Tc3x3FwdHalo {
  static constexpr int BN = BN_;
  // (tap, k16) pairs are dealt round-robin to kIssuers warps, each issuing into
  // its own accumulator copy (summed by the epilogue): eight issuers while the
  // copies fit two CTAs' TMEM, else three
  static constexpr int kIssuers = DPB_FWD_ISSUERS, kAccCopies = kIssuers;
  // producer threads: the warps past the issuers (an issuing warp is held by
  // the tensor pipe's issue rate; the others build the next K chunk meanwhile)
  static constexpr bool kSpecialized = kIssuers < 8;
  static constexpr int kTmemCols = BN * kAccCopies;
  static constexpr bool kTapCols = false;
  static constexpr bool kEarlyPrologue = false;  // BN_b statistics: the predecessor's output
  static constexpr int kMinBlocks = 2;
  static constexpr bool kColSums = true;
  static constexpr bool kBulk = true;
  static constexpr int kEpiPrefetch = 0;  // (see Tc3x3DgradHalo)
  static constexpr bool kKPair = true;  // launched as cluster (1, 2) pairs when kpair
  HaloArgs h;
  // producer threads [prod0, kThreads): past the issuer warps here; all of
  // them for Tc3x3FwdTaps (non-specialised engine path), set by the host
  int prod0 = 32 * kIssuers;
  int raw_want = 2;  // raw ring depth requested by the host (HaloPlan::fwd_ring)
  int kpair = 0;     // 1: CTA (x, y) of a (1, 2) cluster takes K chunks [y * nkb / 2, (y + 1) * nkb / 2)
  __device__ uint32_t halo_bytes() const { return static_cast<uint32_t>(h.g.R * h.kc * 2); }
  __device__ uint32_t b_bytes() const { return static_cast<uint32_t>(9 * BN * h.kc * 2); }
  __device__ uint32_t stage_bytes() const { return 2 * (halo_bytes() + b_bytes()); }
  __device__ int nkb_all() const { return (h.a.bk + h.kc - 1) / h.kc; }
  __device__ int num_kb() const { return kpair ? nkb_all() / 2 : nkb_all(); }
  __device__ int kb0() const { return kpair ? static_cast<int>(blockIdx.y) * (nkb_all() / 2) : 0; }
  __device__ int tile() const { return blockIdx.x % h.g.tpi; }
  __device__ int img() const { return blockIdx.x / h.g.tpi; }
  // aux: BN table | raw fp32 halo ring (depth K chunks) | halo row table.
  // depth 2 fetches chunk kb+1 while kb is transformed; depth 1 (the host's
  // choice when that is what lets two CTAs share an SM) fetches chunk by chunk
  __host__ __device__ static uint32_t raw_offset(int bk) { return (sizeof(BnFwd) * bk + 127) / 128 * 128; }
  __host__ __device__ static uint32_t raw_bytes(int R, int kc) { return static_cast<uint32_t>(R) * kc * 4; }
  __host__ __device__ static int ring_depth(int bk, int kc, int want) {  // one slot when nkb == 1
    const int nkb = (bk + kc - 1) / kc;
    return nkb < want ? nkb : want;
  }
  __host__ __device__ static uint32_t rows_offset(int bk, int R, int kc, int want) {
    return raw_offset(bk) + ring_depth(bk, kc, want) * raw_bytes(R, kc);
  }
  __host__ __device__ static uint32_t aux_bytes(int bk, int R, int kc, int want) {
    return rows_offset(bk, R, kc, want) + 4 * R;
  }
  // K pair: rank 0's exchange buffer [kBM][BN] fp32 after the other tables
  __host__ __device__ static uint32_t xbuf_bytes() { return kBM * BN * 4; }
  __device__ uint32_t xbuf_offset() const { return (aux_bytes(h.a.bk, h.g.R, h.kc, raw_want) + 15) / 16 * 16; }
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(aux), h.a.bk, 0, h.a.bmean, h.a.bvar, h.a.gamma_b,
                h.a.beta_b);
    // halo row r -> element offset of its pixel's z row within the image, or -1 (padding)
    int* rowoff = reinterpret_cast<int*>(aux + rows_offset(h.a.bk, h.g.R, h.kc, raw_want));
    const int t = tile();
    for (int r = threadIdx.x; r < h.g.R; r += kThreads) {
      const int pp = h.g.pixel(h.g.pos(t, r));
      rowoff[r] = pp >= 0 ? pp * h.a.bk : -1;
    }
  }
  __device__ void bulk(uint32_t st, int kb, uint64_t* bar) const {
    mbar_expect_tx(bar, 2 * b_bytes());
    bulk_load(st + 2 * halo_bytes(), h.wt + static_cast<int64_t>(kb0() + kb) * 2 * b_bytes(), 2 * b_bytes(),
              bar);
  }
  // chunk q of a K chunk -> (halo row r, channel offset kk): eight consecutive
  // chunks cover eight rows of one 8-channel group (conflict-free 16-byte
  // stores); shifts when kcn is a power of two (kc = 16, 32, 64), else divisions
  __device__ static void chunk_coords(int q, int kcn, int& r, int& kk) {
    if ((kcn & (kcn - 1)) == 0) {
      const int kcs = __ffs(kcn) - 1;
      r = (q & 7) | ((q >> (3 + kcs)) << 3);
      kk = ((q >> 3) & (kcn - 1)) << 3;
    } else {
      r = (q & 7) + 8 * (q / (8 * kcn));
      kk = ((q >> 3) % kcn) * 8;
    }
  }
  // Raw fp32 halo chunks stream through the ring (cp.async, issued one K chunk
  // ahead): chunk kb+1's loads are in flight while chunk kb is transformed.
  // Each producer thread copies and then transforms the same chunks
  // (thread-local groups: no barrier).
  __device__ void fetch(int kb, uint8_t* aux) const {
    const LayerArgs<float>& a = h.a;
    const int depth = ring_depth(a.bk, h.kc, raw_want);
    const uint32_t ring = smem_u32(aux + raw_offset(a.bk) + (kb % depth) * raw_bytes(h.g.R, h.kc));
    const int* rowoff = reinterpret_cast<const int*>(aux + rows_offset(a.bk, h.g.R, h.kc, raw_want));
    const int kcn = h.kc >> 3;
    const int j_base = (kb0() + kb) * h.kc;
    const float* zb = a.z + static_cast<int64_t>(img()) * h.g.H * h.g.W * a.bk + j_base;
    const int nchunk = h.g.R * kcn;
    const int pthreads = kThreads - prod0;
    for (int q = static_cast<int>(threadIdx.x) - prod0; q < nchunk; q += pthreads) {
      int r, kk;
      chunk_coords(q, kcn, r, kk);
      const int ro = rowoff[r];
      if (ro >= 0 && j_base + kk < a.bk) {
        const float* src = zb + ro + kk;
        cp_async16(ring + q * 32, src);
        cp_async16(ring + q * 32 + 16, src + 4);
      }
    }
    cp_async_commit();
  }
  __device__ void produce(uint8_t* st, int kb, const uint8_t* aux) const {
    if (static_cast<int>(threadIdx.x) < prod0) return;
    const int pthreads = kThreads - prod0;
    const LayerArgs<float>& a = h.a;
    const BnFwd* bn = reinterpret_cast<const BnFwd*>(aux);
    uint8_t* xh = st;
    uint8_t* xl = st + halo_bytes();
    const int nkb = num_kb();
    uint8_t* waux = const_cast<uint8_t*>(aux);
    const int depth = ring_depth(a.bk, h.kc, raw_want);
    if (depth >= 2) {
      if (kb == 0) fetch(0, waux);
      if (kb + 1 < nkb) {  // slot (kb+1) % 2 held chunk kb-1, transformed by this thread already
        fetch(kb + 1, waux);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    } else {  // one slot: this chunk's copies, then its transform
      fetch(kb, waux);
      cp_async_wait<0>();
    }
    const float* ring = reinterpret_cast<const float*>(aux + raw_offset(a.bk) + (kb % depth) * raw_bytes(h.g.R, h.kc));
    const int* rowoff = reinterpret_cast<const int*>(aux + rows_offset(a.bk, h.g.R, h.kc, raw_want));
    const int j_base = (kb0() + kb) * h.kc;
    const int kcn = h.kc >> 3;
    const int nchunk = h.g.R * kcn;
    const int q0 = static_cast<int>(threadIdx.x) - prod0;
    // a thread's channel group is the same for all its chunks when the stride
    // is a multiple of 8 * kcn: its BN constants are loaded once per K chunk
    const bool fixed = (pthreads >> 3) % kcn == 0;
    float mu[8], sc[8], be[8];
    {
      int r0, kk;
      chunk_coords(q0, kcn, r0, kk);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = min(j_base + kk + e, a.bk - 1);
        mu[e] = bn[j].mean;
        sc[e] = bn[j].scale;
        be[e] = bn[j].beta;
      }
    }
    for (int q = q0; q < nchunk; q += pthreads) {
      int r, kk;
      chunk_coords(q, kcn, r, kk);
      const int j0 = j_base + kk;
      const bool ok = rowoff[r] >= 0 && j0 < a.bk;  // false: zero padding (after activation)
      float v[8];
      if (ok) {
        const float4 x0 = *reinterpret_cast<const float4*>(ring + q * 8);
        const float4 x1 = *reinterpret_cast<const float4*>(ring + q * 8 + 4);
        v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
        v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
        if (fixed) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float t = fmaf(v[e] - mu[e], sc[e], be[e]);  // bn_relu
            v[e] = j0 + e < a.bk && t > 0.f ? t : 0.f;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = j0 + e < a.bk ? bn_relu(bn[j0 + e], v[e]) : 0.f;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = 0.f;
      }
      uint4 hi, lo;
      split8_h(v, hi, lo);
      const uint32_t off = halo_kmajor(h.g.R, r, kk);
      st_shared16(xh, off, hi);
      st_shared16(xl, off, lo);
    }
  }
  __device__ void issue(uint32_t st, int kb, uint32_t tmem_base, int part) const {
    constexpr uint32_t idesc = make_idesc(BN, 0, 0, true);
    const uint32_t tmem = tmem_base + part * BN;
    const uint32_t RB = static_cast<uint32_t>(h.g.R) * 16, WB = 9u * BN * 16;
    const uint32_t xh = sdesc_lo(st, RB), xl = sdesc_lo(st + halo_bytes(), RB);
    const uint32_t wh = sdesc_lo(st + 2 * halo_bytes(), WB);
    const uint32_t wl = sdesc_lo(st + 2 * halo_bytes() + b_bytes(), WB);
    const uint32_t hi = sdesc_hi(128);
    const int nk16 = h.kc / 16;  // 9 * nk16 >= 9 pairs: every copy gets at least one
    for (int q = part; q < 9 * nk16; q += kIssuers) {
      const int tap = q / nk16, k16 = q - tap * nk16;
      const uint32_t aoff = static_cast<uint32_t>(h.g.fwd_off(tap));  // 16-byte units
      const uint32_t boff = static_cast<uint32_t>(tap * BN);
      const uint32_t da = aoff + k16 * 2 * (RB >> 4), db = boff + k16 * 2 * (WB >> 4);
      const uint32_t acc = (kb > 0 || q != part) ? 1u : 0u;
      mma_bf16_lh(tmem, xh + da, hi, wh + db, hi, idesc, acc);
      mma_bf16_lh(tmem, xh + da, hi, wl + db, hi, idesc, 1u);
      mma_bf16_lh(tmem, xl + da, hi, wh + db, hi, idesc, 1u);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&s1)[8],
                           float (&s2)[8]) const {
    const LayerArgs<float>& a = h.a;
    const int pp = h.g.pixel(h.g.g_s0(tile()) + row);
    const int nv = pp >= 0 ? a.k - col0 : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool ok = i < nv;
      s1[i] = ok ? v[i] : 0.f;
      s2[i] = ok ? v[i] * v[i] : 0.f;
    }
    if (nv > 0) {
      const int64_t p = static_cast<int64_t>(img()) * h.g.H * h.g.W + pp;
      float* dst = a.feat + p * a.C + a.c + col0;
      if (h.vec && nv >= 8) {
        reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < nv) dst[i] = v[i];
      }
    }
  }
  __device__ void col_sums(int c, double s1, double s2) const {
    if (c < h.a.k) h.a.part[static_cast<int64_t>(blockIdx.x) * h.a.k + c] = make_double2(s1, s2);
  }
};

// Forward with all 9 taps as GEMM columns (k <= 14, k % 4 == 0): B = W2 rows
// tap*k + o (N = 9k padded to 16), A = the whole halo as two M blocks of 128
// rows with no tap shift, so each MMA reads the halo once instead of once per
// tap (the narrow per-tap MMAs are bound by shared-memory operand reads).  The
// engine adds the tap columns at row offsets (kTapCols epilogue).  Produce and
// output epilogue are those of Tc3x3FwdHalo.
struct Tc3x3FwdTaps : Tc3x3FwdHalo<16> {
  static constexpr int kIssuers = 2, kAccCopies = 1;  // one issuer per M block
  static constexpr bool kSpecialized = false;
  static constexpr int kTmemCols = 2 * kBM;           // M block b at columns [128 b, 128 b + N)
  static constexpr bool kTapCols = true;
  static constexpr int kMinBlocks = 2;
  __device__ int np() const { return (9 * h.a.k + 15) / 16 * 16; }
  __device__ uint32_t b_bytes() const { return static_cast<uint32_t>(np() * h.kc * 2); }
  __device__ uint32_t stage_bytes() const { return 2 * (halo_bytes() + b_bytes()); }
  __device__ int tap_k() const { return h.a.k; }
  __device__ int tap_col(int tap) const { return tap * h.a.k; }
  __device__ int tap_off(int tap) const { return h.g.fwd_off(tap); }
  __device__ int rows() const { return h.g.R; }
  __device__ void bulk(uint32_t st, int kb, uint64_t* bar) const {
    mbar_expect_tx(bar, 2 * b_bytes());
    bulk_load(st + 2 * halo_bytes(), h.wt + static_cast<int64_t>(kb) * 2 * b_bytes(), 2 * b_bytes(), bar);
  }
  __device__ void issue(uint32_t st, int kb, uint32_t tmem_base, int part) const {
    const uint32_t idesc = make_idesc(np(), 0, 0, true);
    const uint32_t tmem = tmem_base + part * kBM;
    const uint32_t RB = static_cast<uint32_t>(h.g.R) * 16, WB = static_cast<uint32_t>(np()) * 16;
    const uint32_t xh = sdesc_lo(st, RB), xl = sdesc_lo(st + halo_bytes(), RB);
    const uint32_t wh = sdesc_lo(st + 2 * halo_bytes(), WB);
    const uint32_t wl = sdesc_lo(st + 2 * halo_bytes() + b_bytes(), WB);
    const uint32_t hi = sdesc_hi(128);
    const int nk16 = h.kc / 16;
    for (int k16 = 0; k16 < nk16; ++k16) {
      // rows are 16 bytes apart in the core-matrix layout: M block b starts 128 b rows in
      const uint32_t da = part * kBM + k16 * 2 * (RB >> 4), db = k16 * 2 * (WB >> 4);
      const uint32_t acc = (kb | k16) ? 1u : 0u;
      mma_bf16_lh(tmem, xh + da, hi, wh + db, hi, idesc, acc);
      mma_bf16_lh(tmem, xh + da, hi, wl + db, hi, idesc, 1u);
      mma_bf16_lh(tmem, xl + da, hi, wh + db, hi, idesc, 1u);
    }
  }
};

// W2 for Tc3x3FwdTaps: per K chunk, rows tap*k + o (np rows, zero past 9k),
// K-major, hi plane then lo plane; layer stride `layer_bytes`.
__global__ void k_pretile_w2_taps(const float* __restrict__ params, int c0, int k, int bk, int kc,
                                  int np, int64_t layer_bytes, uint8_t* __restrict__ out) {
  pdl_enter();
  const int l = blockIdx.y;
  int64_t poff = 0;
  for (int j = 0; j < l; ++j) {
    const int cj = c0 + j * k;
    poff += 2LL * cj + static_cast<int64_t>(bk) * cj + 2LL * bk + 9LL * k * bk;
  }
  const int c = c0 + l * k;
  const float* w2 = params + poff + 2 * c + static_cast<int64_t>(bk) * c + 2 * bk;
  const int nkb = (bk + kc - 1) / kc;
  const int plane = np * kc * 2;
  uint8_t* o_l = out + static_cast<int64_t>(l) * layer_bytes;
  const int kcn = kc / 8;
  const int per = np * kcn;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nkb * per; q += gridDim.x * blockDim.x) {
    const int kb = q / per, qq = q - kb * per;
    const int row = qq / kcn, kk = (qq % kcn) * 8;
    const int tap = row / k, o = row - tap * k;
    const int j0 = kb * kc + kk;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = (row < 9 * k && j0 + i < bk) ? w2[(static_cast<int64_t>(o) * bk + j0 + i) * 9 + tap] : 0.f;
    uint4 hh, lo;
    split8_h(v, hh, lo);
    uint8_t* t = o_l + static_cast<int64_t>(kb) * 2 * plane;
    const uint32_t off = halo_kmajor(np, row, kk);
    *reinterpret_cast<uint4*>(t + off) = hh;
    *reinterpret_cast<uint4*>(t + plane + off) = lo;
  }
}

// ---- backward data --------------------------------------------------------------------
// t0[pos][j] = relu'(act_b) * sum_tap sum_o dY[pos - d][o] W2[o][j][tap]; K per
// tap = kc (k padded to 16); the stage holds the dY halo and W2^T for 9 taps.
template <int BN_>
struct Tc3x3DgradHalo {
  static constexpr int BN = BN_;
  // one issuer, one accumulator: the 9 tap MMAs per tile are few, and the
  // small TMEM / register / smem footprint lets three CTAs share an SM, whose
  // phases (halo loads, MMAs, the z-dependent epilogue) then overlap
  static constexpr int kIssuers = 1, kAccCopies = 1;
  static constexpr bool kSpecialized = false;
  static constexpr bool kTapCols = false;
  static constexpr bool kEarlyPrologue = true;  // BN_b forward statistics and parameters
  static constexpr int kMinBlocks = BN <= 64 ? 4 : 2;
  static constexpr int kTmemCols = BN * kAccCopies;
  static constexpr bool kColSums = true;
  static constexpr bool kBulk = true;
  static constexpr int kMaxChunks = 4;
  HaloArgs h;
  __device__ uint32_t halo_bytes() const { return static_cast<uint32_t>(h.g.R * h.kc * 2); }
  __device__ uint32_t b_bytes() const { return static_cast<uint32_t>(9 * BN * h.kc * 2); }
  __device__ uint32_t stage_bytes() const { return halo_bytes() + b_bytes(); }
  __device__ int num_kb() const { return 1; }
  __device__ int tile() const { return blockIdx.x % h.g.tpi; }
  __device__ int img() const { return blockIdx.x / h.g.tpi; }
  __device__ int n0() const { return blockIdx.y * BN; }  // first output column (channel j) of this CTA
  __device__ void prologue(uint8_t* aux) const {
    fill_bn_fwd(reinterpret_cast<BnFwd*>(aux), h.a.bk, 0, h.a.bmean, h.a.bvar, h.a.gamma_b,
                h.a.beta_b);
  }
  __device__ void bulk(uint32_t st, int, uint64_t* bar) const {
    mbar_expect_tx(bar, b_bytes());
    bulk_load(st + halo_bytes(), h.wt + static_cast<int64_t>(blockIdx.y) * b_bytes(), b_bytes(), bar);
  }
  __device__ void produce(uint8_t* st, int, const uint8_t*) const {
    const LayerArgs<float>& a = h.a;
    uint8_t* dy = st;
    const int t = tile();
    const int64_t pix0 = static_cast<int64_t>(img()) * h.g.H * h.g.W;
    const int kcn = h.kc / 8;
    const int nchunk = h.g.R * kcn;
    for (int base = 0; base < nchunk; base += kMaxChunks * kThreads) {
      float v[kMaxChunks][8];
      int rr[kMaxChunks], kk[kMaxChunks];
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        const int q = base + threadIdx.x + i * kThreads;
        rr[i] = (q & 7) + 8 * (q / (8 * kcn));
        kk[i] = ((q >> 3) % kcn) * 8;
        const int pp = q < nchunk ? h.g.pixel(h.g.pos(t, rr[i])) : -1;
        if (pp >= 0 && kk[i] < a.k) load8(a.acc + (pix0 + pp) * a.Ca + a.c + kk[i], a.k - kk[i], h.vec, v[i]);
        else
#pragma unroll
          for (int e = 0; e < 8; ++e) v[i][e] = 0.f;
        if (q >= nchunk) rr[i] = -1;
      }
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i)
        if (rr[i] >= 0) st_shared16(dy, halo_kmajor(h.g.R, rr[i], kk[i]), to_bf16x8(v[i]));
    }
  }
  __device__ void issue(uint32_t st, int, uint32_t tmem_base, int part) const {
    constexpr uint32_t idesc = make_idesc(BN, 0, 0);
    const uint32_t tmem = tmem_base + part * BN;
    const uint32_t RB = static_cast<uint32_t>(h.g.R) * 16, WB = 9u * BN * 16;
    const uint32_t dy = sdesc_lo(st, RB), wt = sdesc_lo(st + halo_bytes(), WB);
    const uint32_t hi = sdesc_hi(128);
    const int nk16 = h.kc / 16;
#pragma unroll
    for (int ti = 0; ti < 9 / kIssuers; ++ti) {
      const int tap = part + kIssuers * ti;
      const uint32_t aoff = static_cast<uint32_t>(h.g.bwd_off(tap));
      const uint32_t boff = static_cast<uint32_t>(tap * BN);
#pragma unroll
      for (int k16 = 0; k16 < 4; ++k16) {
        if (k16 >= nk16) break;
        mma_bf16_lh(tmem, dy + aoff + k16 * 2 * (RB >> 4), hi, wt + boff + k16 * 2 * (WB >> 4), hi,
                    idesc, (ti | k16) ? 1u : 0u);
      }
    }
  }
  static constexpr int kEpiPrefetch = BN <= 64 ? 2 : 4;  // z column groups per load batch (register cap)
  static constexpr bool kKPair = false;
  __device__ void epi_load(int row, int col0, float (&zv)[8]) const {
    const LayerArgs<float>& a = h.a;
    col0 += n0();
    const int pp = h.g.pixel(h.g.g_s0(tile()) + row);
    const int nv = pp >= 0 ? a.bk - col0 : 0;
    const int64_t p = static_cast<int64_t>(img()) * h.g.H * h.g.W + (pp >= 0 ? pp : 0);
#ifdef DPB_EXP_NOZ
    for (int i = 0; i < 8; ++i) zv[i] = 1.f + row * 1e-3f;
#else
    if (nv > 0) load8(a.z + p * a.bk + col0, nv, (a.bk & 3) == 0, zv);
#endif
  }
  __device__ void epilogue(int, int, const float (&)[8], const uint8_t*, float (&)[8], float (&)[8]) const {}
  __device__ void epilogue_pre(int row, int col0, const float (&v)[8], const uint8_t* aux, const float (&zv)[8],
                               float (&s1)[8], float (&s2)[8]) const {
    const LayerArgs<float>& a = h.a;
    const BnFwd* bn = reinterpret_cast<const BnFwd*>(aux);
    col0 += n0();
    const int pp = h.g.pixel(h.g.g_s0(tile()) + row);
    const int nv = pp >= 0 ? a.bk - col0 : 0;
    float g[8];
    const int64_t p = static_cast<int64_t>(img()) * h.g.H * h.g.W + (pp >= 0 ? pp : 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < nv) {
        const BnFwd b = bn[col0 + i];
        g[i] = relu_mask_ref(b, zv[i]) ? v[i] : 0.f;
        s1[i] = g[i];
        s2[i] = g[i] * ((zv[i] - b.mean) * b.inv);
      } else {
        g[i] = 0.f;
        s1[i] = 0.f;
        s2[i] = 0.f;
      }
    }
#ifdef DPB_EXP_NOSTORE
    if (false) {
#else
    if (nv > 0) {
#endif
      float* dst = a.g0 + p * a.bk + col0;
      if ((a.bk & 3) == 0 && nv >= 8) {
        reinterpret_cast<float4*>(dst)[0] = make_float4(g[0], g[1], g[2], g[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(g[4], g[5], g[6], g[7]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < nv) dst[i] = g[i];
      }
    }
  }
  __device__ void col_sums(int c, double s1, double s2) const {
    if (n0() + c < h.a.bk) h.a.part[static_cast<int64_t>(blockIdx.x) * h.a.bk + n0() + c] = make_double2(s1, s2);
  }
};

// ---- backward weights ------------------------------------------------------------------
// CTA (x, y): tiles [x*tpc, (x+1)*tpc) of the global tile list (all images),
// channels j in [128*y, 128*y + 128).  Per tile the stage holds act_b's halo
// (MN-major: rows = channels, K = positions) and dY of the tile's 128
// positions (MN-major: rows = o).  Tap t accumulates into TMEM columns
// [t*BN, t*BN + BN).
template <int BN_>
struct Tc3x3WgradHalo {
  static constexpr int BN = BN_;
  static constexpr int kIssuers = 3, kAccCopies = 1;  // taps t = warp, warp+3, warp+6
  static constexpr bool kSpecialized = false;
  static constexpr bool kTapCols = false;
  static constexpr bool kEarlyPrologue = true;  // BN_b forward statistics and parameters
  static constexpr int kMinBlocks = 2;
  static constexpr int kTmemCols = 9 * BN;
  static constexpr bool kColSums = false;
  static constexpr bool kBulk = false;
  static constexpr int kEpiPrefetch = 0;  // (see Tc3x3DgradHalo)
  static constexpr bool kKPair = false;
  static constexpr int kMaxChunks = 6;  // bk = 48 at W = 32: 1456 chunks, one load batch
  HaloArgs h;
  int tpc;      // tiles per CTA
  int ntiles;   // total tiles = N * tpi
  __device__ uint32_t halo_bytes() const { return static_cast<uint32_t>(h.g.R * kBM * 2); }
  __device__ uint32_t b_bytes() const { return static_cast<uint32_t>(kBM * BN * 2); }
  __device__ uint32_t stage_bytes() const { return halo_bytes() + b_bytes(); }
  __device__ int num_kb() const {
    const int t0 = blockIdx.x * tpc;
    const int n = ntiles - t0;
    return n < 0 ? 0 : (n < tpc ? n : tpc);
  }
  // aux: BN table as float4 {mean, scale, beta, -} | two halo row tables
  // (stage parity): row r -> image-local pixel of the tile's halo row, or -1
  __host__ __device__ static uint32_t rows_offset(int bk) { return (16 * bk + 127) / 128 * 128; }
  __host__ __device__ static uint32_t aux_bytes(int bk, int R) { return rows_offset(bk) + 2 * 4 * R; }
  // halo row table of K block kb (the CTA's kb-th tile) into table kb & 1:
  // the prologue fills table 0, produce(kb) fills table kb+1 after its own
  // loads, so no extra barrier (the engine's barrier after produce orders it)
  __device__ void fill_rows(const uint8_t* aux, int kb) const {
    int* rows = const_cast<int*>(reinterpret_cast<const int*>(aux + rows_offset(h.a.bk))) + (kb & 1) * h.g.R;
    const int gt = blockIdx.x * tpc + kb;
    const int t = gt - (gt / h.g.tpi) * h.g.tpi;
    for (int r = threadIdx.x; r < h.g.R; r += kThreads) rows[r] = h.g.pixel(h.g.pos(t, r));
  }
  __device__ void prologue(uint8_t* aux) const {
    float4* bq = reinterpret_cast<float4*>(aux);
    for (int j = threadIdx.x; j < h.a.bk; j += kThreads) {
      const float inv = bn_inv(h.a.bvar[j]);
      bq[j] = make_float4(h.a.bmean[j], h.a.gamma_b[j] * inv, h.a.beta_b[j], 0.f);  // fill_bn_fwd's fields
    }
    fill_rows(aux, 0);
  }
  __device__ void bulk(uint32_t, int, uint64_t*) const {}
  __device__ void produce(uint8_t* st, int kb, const uint8_t* aux) const {
    const LayerArgs<float>& a = h.a;
    const float4* bq = reinterpret_cast<const float4*>(aux);
    int* rows = const_cast<int*>(reinterpret_cast<const int*>(aux + rows_offset(a.bk))) + (kb & 1) * h.g.R;
    uint8_t* xs = st;
    uint8_t* dys = st + halo_bytes();
    const int gt = blockIdx.x * tpc + kb;
    const int im = gt / h.g.tpi;
    const float* zb = a.z + static_cast<int64_t>(im) * h.g.H * h.g.W * a.bk;
    const float* gb = a.acc + static_cast<int64_t>(im) * h.g.H * h.g.W * a.Ca + a.c;
    const int j_base = blockIdx.y * kBM;
    // only the channel groups below bk: the A rows j >= bk feed only D rows the
    // epilogue drops (an MMA row depends on its own A row), so they stay unwritten
    const int jn = a.bk - j_base < kBM ? a.bk - j_base : kBM;
    const int groups = (jn + 7) / 8;
    const bool gp2 = (groups & (groups - 1)) == 0;
    const int gs = __ffs(groups) - 1;
    const int nchunk = h.g.R * groups;  // act_b halo chunks; then dY chunks
    const int og = BN / 8;
    const int ndy = kBM * og;
    const int dy0 = h.g.W2 + 1;  // halo row of the tile's first output position
    const int total = nchunk + ndy;
    for (int base = 0; base < total; base += kMaxChunks * kThreads) {
      float v[kMaxChunks][8];
      uint32_t off[kMaxChunks];
      uint8_t kind[kMaxChunks];  // 0 skip, 1 halo, 2 dY, 3 zero
      int jj[kMaxChunks];
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        const int q = base + threadIdx.x + i * kThreads;
        kind[i] = 0;
        jj[i] = 0;
        off[i] = 0;
        if (q < nchunk) {
          // act_b halo, MN-major: phase = 8 consecutive positions of one group
          const int pos = gp2 ? ((q & 7) | ((q >> (3 + gs)) << 3)) : (q & 7) + 8 * (q / (8 * groups));
          const int jg = gp2 ? ((q >> 3) & (groups - 1)) << 3 : ((q >> 3) % groups) * 8;
          const int j0 = j_base + jg;
          const int pp = rows[pos];
          const bool valid = pp >= 0 && j0 < a.bk;
          if (valid) load8(zb + static_cast<int64_t>(pp) * a.bk + j0, a.bk - j0, (a.bk & 3) == 0, v[i]);
          kind[i] = valid ? 1 : 3;  // 3: zero padding (after activation)
          jj[i] = j0;
          off[i] = halo_mnmajor(h.g.R, jg, pos);
        } else if (q < total) {
          const int r = q - nchunk;
          const int pos = (r & 7) + 8 * (r / (8 * og));
          const int o0 = ((r >> 3) % og) * 8;
          const int pp = rows[dy0 + pos];
          if (pp >= 0 && o0 < a.k) load8(gb + static_cast<int64_t>(pp) * a.Ca + o0, a.k - o0, h.vec, v[i]);
          else
#pragma unroll
            for (int e = 0; e < 8; ++e) v[i][e] = 0.f;
          kind[i] = 2;
          off[i] = halo_mnmajor(kBM, o0, pos);
        }
      }
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        if (kind[i] == 1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 b = bq[min(jj[i] + e, a.bk - 1)];
            const float tt = fmaf(v[i][e] - b.x, b.y, b.z);  // bn_relu
            v[i][e] = jj[i] + e < a.bk && tt > 0.f ? tt : 0.f;
          }
          st_shared16(xs, off[i], to_bf16x8(v[i]));
        } else if (kind[i] == 2) {
          st_shared16(dys, off[i], to_bf16x8(v[i]));
        } else if (kind[i] == 3) {
          st_shared16(xs, off[i], make_uint4(0, 0, 0, 0));
        }
      }
    }
    if (kb + 1 < num_kb()) fill_rows(aux, kb + 1);
  }
  __device__ void issue(uint32_t st, int kb, uint32_t tmem, int part) const {
    constexpr uint32_t idesc = make_idesc(BN, 1, 1);
    const uint32_t RB = static_cast<uint32_t>(h.g.R) * 16;
    // A: M = channels (SBO = R*16 between channel groups), K = positions
    // shifted by the tap (LBO = 128 between groups of 8 positions)
    const uint32_t xs = sdesc_lo(st, 128), dys = sdesc_lo(st + halo_bytes(), 128);
    const uint32_t ahi = sdesc_hi(RB), bhi = sdesc_hi(kBM * 16);
#pragma unroll
    for (int ti = 0; ti < 3; ++ti) {
      const int tap = part + 3 * ti;
      const uint32_t aoff = static_cast<uint32_t>(h.g.fwd_off(tap));
#pragma unroll
      for (int k16 = 0; k16 < kBM / 16; ++k16)
        mma_bf16_lh(tmem + tap * BN, xs + aoff + k16 * 16, ahi, dys + k16 * 16, bhi, idesc,
                    (kb | k16) ? 1u : 0u);
    }
  }
  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*, float (&)[8],
                           float (&)[8]) const {
    const LayerArgs<float>& a = h.a;
    const int tap = col0 / BN, o0 = col0 - tap * BN;
    const int j = blockIdx.y * kBM + row;
    const int nv = j < a.bk ? a.k - o0 : 0;
    float* dst = a.wpart + (static_cast<int64_t>(blockIdx.x) * 9 * a.bk + tap * a.bk + j) * a.k + o0;
    if ((a.k & 3) == 0 && nv >= 4) {  // rows of k floats, o0 % 8 == 0: 16-byte aligned quads
      reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
      if (nv >= 8) reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
      else
#pragma unroll
        for (int i = 4; i < 8; ++i)
          if (i < nv) dst[i] = v[i];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < nv) dst[i] = v[i];
    }
  }
  __device__ void col_sums(int, double, double) const {}
};

}  // namespace tc
}  // namespace dpb
