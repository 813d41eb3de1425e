// tcgen05 (5th-gen tensor core) implicit-GEMM engine for sm_100a.
//
// One CTA computes a 128 x BN fp32 tile of D = A . B^T in TMEM:
//   * all 256 threads are producers: they load the op's operands from HBM,
//     apply the fused transform (BN+ReLU recompute, 3x3 halo gather with
//     zero padding after activation, BN-backward), convert to bf16 — for the
//     forward as an exact hi/lo split, x = hi + lo — and st.shared them into
//     the UMMA canonical no-swizzle layout (8x8 core matrices), double
//     buffered;
//   * one elected thread issues tcgen05.mma (kind::f16, bf16 x bf16 -> fp32,
//     M=128) and tcgen05.commit's each stage to an mbarrier, so the tensor
//     core runs stage s while the producers fill stage s^1;
//   * the epilogue reads the accumulator with tcgen05.ld (32x32b) and hands
//     8-column chunks of each row to the op (stores, ReLU masks, BN sums).
//
// Forward GEMMs run as bf16x3 (hi.hi + hi.lo + lo.hi, fp32 accumulate):
// ~16 mantissa bits per operand, enough that ReLU masks match the fp32
// reference; backward GEMMs use one bf16 product.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "dpb_common.cuh"

namespace dpb {
namespace tc {

constexpr int kBM = 128;   // UMMA M (cta_group::1)
constexpr int kBK = 64;    // K elements per pipeline stage (4 MMAs of K=16)
constexpr int kThreads = 256;

// ---- PTX wrappers --------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---- thread-block clusters (DSMEM) ----------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address -> the same offset in CTA `rank`'s shared memory (shared::cluster)
__device__ __forceinline__ uint32_t mapa_cluster(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
// every thread of every CTA in the cluster: release this CTA's writes, acquire the others'
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

// D[tmem] (+)= A[smem] . B[smem]^T, bf16 inputs, fp32 accumulate.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Same MMA with the two descriptors given as 32-bit halves (the hot issue
// loops only add byte offsets to the low halves).
__device__ __forceinline__ void mma_bf16_lh(uint32_t d_tmem, uint32_t alo, uint32_t ahi,
                                            uint32_t blo, uint32_t bhi, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      ".reg .b64 da, db;\n"
      "mov.b64 da, {%1, %2};\n"
      "mov.b64 db, {%3, %4};\n"
      "setp.ne.b32 p, %6, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(accumulate));
}

// Low / high 32 bits of a no-swizzle smem descriptor; adding (bytes >> 4) to
// the low half moves the start address.
// Warp-collective forms: every lane of a convergent warp executes them with
// warp-uniform operands and one elected lane issues, so the compiler keeps the
// descriptors in uniform registers (no per-MMA R2UR waterfall).
__device__ __forceinline__ void mma_bf16_lh_w(uint32_t d_tmem, uint32_t alo, uint32_t ahi,
                                              uint32_t blo, uint32_t bhi, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b64 da, db;\n"
      "mov.b64 da, {%1, %2};\n"
      "mov.b64 db, {%3, %4};\n"
      "setp.ne.b32 p, %6, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// warp-uniform copy of a value every lane holds
__device__ __forceinline__ uint32_t uniform(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

__device__ __forceinline__ uint32_t sdesc_lo(uint32_t saddr, uint32_t lbo) {
  return ((saddr >> 4) & 0x3FFF) | (((lbo >> 4) & 0x3FFF) << 16);
}
__device__ __forceinline__ uint32_t sdesc_hi(uint32_t sbo) {
  return ((sbo >> 4) & 0x3FFF) | (1u << 14);  // version 1 at bit 46
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bits, 8 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 4 consecutive TMEM columns of this warp's 32 lanes (no wait: tmem_wait_ld).
__device__ __forceinline__ void tmem_ld4_nowait(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 16 consecutive TMEM columns of this warp's 32 lanes (one wait).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 consecutive TMEM columns of this warp's 32 lanes (one wait).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
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

// ---- async-copy / barrier PTX (mbarrier tx counts, TMA, bulk copies) ---------
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// TMA tile store smem -> global (bulk async group; out-of-bounds parts clipped).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed bulk groups still READ shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Ampere-style asynchronous 16-byte global -> shared copies (per-thread groups).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(reinterpret_cast<uint64_t>(src))
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- descriptors -----------------------------------------------------------------

// Instruction descriptor: bf16 A/B, fp32 D, M=128, N, majors (0 = K, 1 = MN).
// kind::f16 operand formats: BF16 (1) by default; f16 = true selects F16 (0),
// the forward GEMMs' fp16x3 split (below).
__host__ __device__ constexpr uint32_t make_idesc(int n, int a_mn, int b_mn, bool f16 = false) {
  return (1u << 4)                                   // D format F32
         | ((f16 ? 0u : 1u) << 7)                    // A format F16 / BF16
         | ((f16 ? 0u : 1u) << 10)                   // B format F16 / BF16
         | (static_cast<uint32_t>(a_mn) << 15)       // A major
         | (static_cast<uint32_t>(b_mn) << 16)       // B major
         | (static_cast<uint32_t>(n >> 3) << 17)     // N >> 3
         | (static_cast<uint32_t>(kBM >> 4) << 24);  // M >> 4
}

// Shared-memory descriptor, SWIZZLE_NONE canonical layout, version 1.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Operand tile of R rows (M or N) x kBK K-elements, bf16, 8x8 core matrices.
// Core matrix (g = row/8, kg = k/8) lives at ((kg * R/8) + g) * 128 bytes.
//   K-major : element (row, k) at core + (row%8)*16 + (k%8)*2
//   MN-major: element (row, k) at core + (k%8)*16 + (row%8)*2
// For both: SBO (next 8 rows along M/N) = 128 B, LBO (next 8 along K) = R*16 B.
template <int R>
struct Tile {
  static constexpr int kBytes = R * kBK * 2;
  // byte offset of the 16-byte chunk holding 8 K-consecutive elements of a row
  // (K-major) starting at k (k % 8 == 0)
  __device__ static constexpr uint32_t kmajor_chunk(int row, int k) {
    return static_cast<uint32_t>(((k >> 3) * (R >> 3) + (row >> 3)) * 128 + (row & 7) * 16);
  }
  // byte offset of the 16-byte chunk holding 8 row-consecutive elements at one
  // k (MN-major), row % 8 == 0
  __device__ static constexpr uint32_t mnmajor_chunk(int row, int k) {
    return static_cast<uint32_t>(((k >> 3) * (R >> 3) + (row >> 3)) * 128 + (k & 7) * 16);
  }
  __device__ static uint64_t desc(uint32_t base, int k16) {
    return make_sdesc(base + static_cast<uint32_t>(k16 * 2 * (R >> 3) * 128), R * 16, 128);
  }
};

// Producer chunk coordinates.  A warp's 128-bit shared stores execute in four
// phases of 8 threads; these mappings give each phase one whole 128-byte core
// matrix (8 rows of one K chunk, or 8 K-rows of one row group), so the stores
// are bank-conflict free.
// K-major: chunk q -> (row, kc), kc a multiple of 8.
__device__ __forceinline__ void kmajor_coords(int q, int& row, int& kc) {
  row = (q & 7) | ((q >> 6) << 3);
  kc = ((q >> 3) & 7) << 3;
}
// MN-major over R rows: chunk q -> (row0, k), row0 a multiple of 8.
template <int R>
__device__ __forceinline__ void mnmajor_coords(int q, int& row0, int& k) {
  const int rest = q >> 3;
  row0 = (rest % (R / 8)) << 3;
  k = ((rest / (R / 8)) << 3) | (q & 7);
}

// ---- bf16 conversion helpers -----------------------------------------------------

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// hi = bf16(x), lo = bf16(x - hi): x == hi + lo to ~16 mantissa bits.
__device__ __forceinline__ void split8(const float (&v)[8], uint4& hi, uint4& lo) {
  float h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    h[i] = __bfloat162float(__float2bfloat16_rn(v[i]));
    l[i] = v[i] - h[i];
  }
  hi = make_uint4(pack_bf16(h[0], h[1]), pack_bf16(h[2], h[3]), pack_bf16(h[4], h[5]),
                  pack_bf16(h[6], h[7]));
  lo = make_uint4(pack_bf16(l[0], l[1]), pack_bf16(l[2], l[3]), pack_bf16(l[4], l[5]),
                  pack_bf16(l[6], l[7]));
}

// Fast exact split for the bf16x3 operands: hi = x with the low 16 mantissa
// bits cleared (exact), lo = bf16_rn(x - hi) (x - hi is exact in fp32), so
// hi + lo == x to 2^-16 relative; two elements packed per instruction.
__device__ __forceinline__ void split8_fast(const float (&v)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = __float_as_uint(v[2 * i]), b = __float_as_uint(v[2 * i + 1]);
    h[i] = __byte_perm(a, b, 0x7632);  // upper halves: a -> low 16 bits, b -> high
    const float ra = v[2 * i] - __uint_as_float(a & 0xFFFF0000u);
    const float rb = v[2 * i + 1] - __uint_as_float(b & 0xFFFF0000u);
    l[i] = pack_bf16(ra, rb);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Forward-GEMM operand split (fp16x3): hi = fp16_rn(x), lo = fp16_rn(x - hi),
// so hi + lo == x to 2^-22 relative (11 + 11 significant bits) for |x| in
// fp16's normal range; lo in the subnormals costs at most 2^-25 absolute.
// Products hi.hi + hi.lo + lo.hi (kind::f16, F16 operands, fp32 accumulate)
// carry ~21 bits, against ~16 for a bf16 hi/lo split: through 264 layers the
// forward's rounding flips ReLU masks, and each flip moves a gradient by O(1)
// (DESIGN.md 2), so the forward's precision sets the gradients' error.  The
// activations (BN+ReLU outputs) and weights are far inside fp16's range.
__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void split8_h(const float (&v)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 hh = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    const float2 f = __half22float2(hh);
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = pack_f16(v[2 * i] - f.x, v[2 * i + 1] - f.y);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ uint4 to_bf16x8(const float (&v)[8]) {
  return make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                    pack_bf16(v[6], v[7]));
}

__device__ __forceinline__ void st_shared16(uint8_t* base, uint32_t off, uint4 v) {
  *reinterpret_cast<uint4*>(base + off) = v;
}

__device__ __forceinline__ void zero8(float (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 0.f;
}

__device__ __forceinline__ void store8(float* p, int n, bool aligned, const float (&v)[8]) {
  if (aligned && n >= 8) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < n) p[i] = v[i];
  }
}

// 8 consecutive fp32 values, vectorised when 16-byte aligned, zero past `n`.
__device__ __forceinline__ void load8(const float* p, int n, bool aligned, float (&v)[8]) {
  if (aligned && n >= 8) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < n ? __ldg(p + i) : 0.f;
  }
}

// ---- the engine ---------------------------------------------------------------------
//
// Op interface (all device functions, called by every thread unless noted):
//   static constexpr int BN;            N tile (multiple of 16, <= 256)
//   static constexpr bool kSplit;       hi/lo operand planes, three MMAs per K step
//   static constexpr bool kF16;         F16 operands (the forward's fp16x3) instead of BF16
//   static constexpr int kAMN, kBMN;    operand majors (0 K-major, 1 MN-major)
//   int num_kb() const;                 K blocks of kBK
//   void prologue(uint8_t* aux) const;  fill coefficient tables
//   void produce(uint8_t* a_hi, uint8_t* a_lo, uint8_t* b_hi, uint8_t* b_lo,
//                int kb, const uint8_t* aux) const;
//   void epilogue(int row, int col0, const float (&v)[8], const uint8_t* aux,
//                 float (&s1)[8], float (&s2)[8]) const;   8 columns of one row
//   void col_sums(int col, float s1, float s2) const;     once per column per CTA
//                                                         (when kColSums)
// TMEM columns to allocate for N accumulator columns (a power of two >= 32).
template <int N>
struct TmemCols {
  static_assert(N >= 1 && N <= 512, "TMEM holds at most 512 fp32 columns per SM");
  static constexpr uint32_t value =
      N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : N <= 256 ? 256 : 512;
};

template <class Op>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const Op op) {
  constexpr int BN = Op::BN;
  constexpr int NP = Op::kSplit ? 2 : 1;  // operand planes
  constexpr int A_BYTES = Tile<kBM>::kBytes;
  constexpr int B_BYTES = Tile<BN>::kBytes;
  constexpr int STAGE = NP * (A_BYTES + B_BYTES);
  constexpr uint32_t TCOLS = TmemCols<BN>::value;
  static_assert(BN % 16 == 0 && BN <= 256, "UMMA N");

  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  __shared__ float red[2][4][BN];

  const int tid = threadIdx.x;
  const int warp = tid / 32, lane = tid % 32;
  uint8_t* aux = smem + 2 * STAGE;

  if (warp == 0) tmem_alloc<TCOLS>(&tmem_base);
  if (tid == 32) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_barrier_init();
  }
  pdl_enter();  // barrier init / TMEM alloc above overlap the predecessor
  op.prologue(aux);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  constexpr uint32_t idesc = make_idesc(BN, Op::kAMN, Op::kBMN, Op::kF16);
  const int nkb = op.num_kb();
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb & 1;
    if (kb >= 2) mbar_wait(&mbar[s], ((kb - 2) >> 1) & 1);  // stage s free again
    uint8_t* st = smem + s * STAGE;
    uint8_t* a_hi = st;
    uint8_t* b_hi = st + A_BYTES;
    uint8_t* a_lo = st + A_BYTES + B_BYTES;
    uint8_t* b_lo = a_lo + A_BYTES;
    op.produce(a_hi, a_lo, b_hi, b_lo, kb, aux);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t ah = smem_u32(a_hi), bh = smem_u32(b_hi);
      const uint32_t al = smem_u32(a_lo), bl = smem_u32(b_lo);
#pragma unroll
      for (int k16 = 0; k16 < kBK / 16; ++k16) {
        const uint32_t acc = (kb | k16) ? 1u : 0u;
        mma_bf16(tmem, Tile<kBM>::desc(ah, k16), Tile<BN>::desc(bh, k16), idesc, acc);
        if constexpr (Op::kSplit) {
          mma_bf16(tmem, Tile<kBM>::desc(ah, k16), Tile<BN>::desc(bl, k16), idesc, 1u);
          mma_bf16(tmem, Tile<kBM>::desc(al, k16), Tile<BN>::desc(bh, k16), idesc, 1u);
        }
      }
      mma_commit(&mbar[s]);
    }
  }
  // wait for the last commit (it covers every earlier MMA of this thread)
  mbar_wait(&mbar[(nkb - 1) & 1], ((nkb - 1) >> 1) & 1);
  tc_fence_after();

  // epilogue: warp w reads TMEM lanes 32*(w%4).. (its quarter), chunks of 8
  // columns split between the two warps of each quarter.
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  for (int cc = half; cc < BN / 8; cc += 2) {
    float v[8];
    tmem_ld8(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cc * 8, v);
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
  tc_fence_before();
  __syncthreads();
  if constexpr (Op::kColSums) {
    for (int c = tid; c < BN; c += kThreads) {
      // fixed order over the four row quarters: deterministic
      const double a = static_cast<double>(red[0][0][c]) + red[0][1][c] + red[0][2][c] + red[0][3][c];
      const double b = static_cast<double>(red[1][0][c]) + red[1][1][c] + red[1][2][c] + red[1][3][c];
      op.col_sums(c, a, b);
    }
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<TCOLS>(tmem);
  }
}

// Dynamic shared memory of the two pipeline stages (the op's aux tables
// follow them).
template <class Op>
constexpr size_t stage_bytes() {
  constexpr int NP = Op::kSplit ? 2 : 1;
  return 2 * NP * (Tile<kBM>::kBytes + Tile<Op::BN>::kBytes);
}

}  // namespace tc
}  // namespace dpb
