// Self-test of the tcgen05 engine: plain D = A . B^T from fp32 global
// operands, every operand major and the bf16x3 split, checked by
// tests/test_tc_gpu.py against an fp64 host GEMM.  Diagnostic entry point
// dpb_selftest_tc_gemm (include/dpb.h).
#include <cuda_runtime.h>

#include "../../include/dpb.h"
#include "dpb_internal.h"
#include "dpb_tc.cuh"

namespace dpb {
namespace tc {

template <int BN_, int AMN, int BMN, bool SPLIT>
struct TestGemm {
  static constexpr int BN = BN_;
  static constexpr bool kSplit = SPLIT;
  static constexpr bool kF16 = false;  // the engine diagnostic keeps bf16 (x3) operands
  static constexpr int kAMN = AMN, kBMN = BMN;
  static constexpr bool kColSums = true;
  const float* A;  // K-major: [M][K]; MN-major: [K][M]
  const float* B;  // K-major: [N][K]; MN-major: [K][N]
  float* D;        // [M][N]
  float* colsum;   // [gridDim.x][N] (sum, sum of squares)
  int M, N, K;

  __device__ int num_kb() const { return (K + kBK - 1) / kBK; }
  __device__ void prologue(uint8_t*) const {}

  template <int R, int MN>
  __device__ void produce_tile(const float* G, int rows_total, int r0, int k0, uint8_t* hi,
                               uint8_t* lo) const {
    for (int q = threadIdx.x; q < R * kBK / 8; q += kThreads) {
      float v[8];
      uint32_t off;
      if (MN == 0) {
        int row, kc;
        kmajor_coords(q, row, kc);
        const int gr = r0 + row, gk = k0 + kc;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = (gr < rows_total && gk + i < K) ? G[static_cast<int64_t>(gr) * K + gk + i] : 0.f;
        off = Tile<R>::kmajor_chunk(row, kc);
      } else {
        int rg, kr;
        mnmajor_coords<R>(q, rg, kr);
        const int gk = k0 + kr;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = (gk < K && r0 + rg + i < rows_total)
                     ? G[static_cast<int64_t>(gk) * rows_total + r0 + rg + i]
                     : 0.f;
        off = Tile<R>::mnmajor_chunk(rg, kr);
      }
      if (kSplit) {
        uint4 h, l;
        split8(v, h, l);
        st_shared16(hi, off, h);
        st_shared16(lo, off, l);
      } else {
        st_shared16(hi, off, to_bf16x8(v));
      }
    }
  }

  __device__ void produce(uint8_t* a_hi, uint8_t* a_lo, uint8_t* b_hi, uint8_t* b_lo, int kb,
                          const uint8_t*) const {
    produce_tile<kBM, AMN>(A, M, blockIdx.x * kBM, kb * kBK, a_hi, a_lo);
    produce_tile<BN, BMN>(B, N, blockIdx.y * BN, kb * kBK, b_hi, b_lo);
  }

  __device__ void epilogue(int row, int col0, const float (&v)[8], const uint8_t*,
                           float (&s1)[8], float (&s2)[8]) const {
    const int gr = blockIdx.x * kBM + row;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gc = blockIdx.y * BN + col0 + i;
      const bool ok = gr < M && gc < N;
      if (ok) D[static_cast<int64_t>(gr) * N + gc] = v[i];
      s1[i] = ok ? v[i] : 0.f;
      s2[i] = ok ? v[i] * v[i] : 0.f;
    }
  }

  __device__ void col_sums(int c, double a, double b) const {
    const int gc = blockIdx.y * BN + c;
    if (gc < N) {
      colsum[(static_cast<int64_t>(blockIdx.x) * N + gc) * 2] = static_cast<float>(a);
      colsum[(static_cast<int64_t>(blockIdx.x) * N + gc) * 2 + 1] = static_cast<float>(b);
    }
  }
};

template <int BN, int AMN, int BMN, bool SPLIT>
static int run(const float* A, const float* B, float* D, float* cs, int M, int N, int K,
               cudaStream_t st) {
  using Op = TestGemm<BN, AMN, BMN, SPLIT>;
  Op op{A, B, D, cs, M, N, K};
  const size_t sm = stage_bytes<Op>();
  cudaFuncSetAttribute(tc_gemm_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(sm));
  dim3 grid((M + kBM - 1) / kBM, (N + BN - 1) / BN);
  tc_gemm_kernel<Op><<<grid, kThreads, sm, st>>>(op);
  return cudaGetLastError();
}

template <int BN>
static int dispatch_major(const float* A, const float* B, float* D, float* cs, int M, int N,
                          int K, int amn, int bmn, int split, cudaStream_t st) {
  const int code = amn * 4 + bmn * 2 + split;
  switch (code) {
    case 0: return run<BN, 0, 0, false>(A, B, D, cs, M, N, K, st);
    case 1: return run<BN, 0, 0, true>(A, B, D, cs, M, N, K, st);
    case 2: return run<BN, 0, 1, false>(A, B, D, cs, M, N, K, st);
    case 3: return run<BN, 0, 1, true>(A, B, D, cs, M, N, K, st);
    case 4: return run<BN, 1, 0, false>(A, B, D, cs, M, N, K, st);
    case 5: return run<BN, 1, 0, true>(A, B, D, cs, M, N, K, st);
    case 6: return run<BN, 1, 1, false>(A, B, D, cs, M, N, K, st);
    default: return run<BN, 1, 1, true>(A, B, D, cs, M, N, K, st);
  }
}

}  // namespace tc
}  // namespace dpb

extern "C" int dpb_selftest_tc_gemm(const float* A, const float* B, float* D, float* colsum,
                                    int M, int N, int K, int bn, int a_mn, int b_mn, int split,
                                    void* stream) {
  using namespace dpb::tc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int e;
  switch (bn) {
    case 16: e = dispatch_major<16>(A, B, D, colsum, M, N, K, a_mn, b_mn, split, st); break;
    case 48: e = dispatch_major<48>(A, B, D, colsum, M, N, K, a_mn, b_mn, split, st); break;
    case 64: e = dispatch_major<64>(A, B, D, colsum, M, N, K, a_mn, b_mn, split, st); break;
    case 128: e = dispatch_major<128>(A, B, D, colsum, M, N, K, a_mn, b_mn, split, st); break;
    case 192: e = dispatch_major<192>(A, B, D, colsum, M, N, K, a_mn, b_mn, split, st); break;
    default: return dpb::fail(DPB_CONFIG_ERROR, "selftest bn must be 16/48/64/128/192");
  }
  if (e != 0) return dpb::cuda_fail(static_cast<cudaError_t>(e), "tc selftest launch");
  return DPB_OK;
}
