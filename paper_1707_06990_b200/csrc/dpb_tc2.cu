// Launchers of the persistent TMA-fed engine (dpb_tc2.cuh) and the host-side
// TMA tensor-map encoding (driver entry point cuTensorMapEncodeTiled).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "dpb_internal.h"
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
static void launch2(Block* b, const Op& op, int ntiles, size_t aux) {
  static bool configured = false;
  if (!configured) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, tc2::tc2_kernel<Op>);
    cudaFuncSetAttribute(tc2::tc2_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024 - static_cast<int>(fa.sharedSizeBytes));
    configured = true;
  }
  const size_t smem = 1024 + Op::kNR * Op::kRawBytes + Op::kNS * Op::kOpBytes + aux;
  const int grid = std::min(ntiles, num_sms());
  tc2::tc2_kernel<Op><<<grid, tc2::kThreads, smem, b->stream>>>(op);
}

template <class Op>
static constexpr size_t fixed_smem() {
  return 1024 + Op::kNR * Op::kRawBytes + Op::kNS * Op::kOpBytes;
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
    case 16: tc2::k_pretile_w1_all<16><<<grid, 256, 0, b->stream>>>(params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 32: tc2::k_pretile_w1_all<32><<<grid, 256, 0, b->stream>>>(params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 48: tc2::k_pretile_w1_all<48><<<grid, 256, 0, b->stream>>>(params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 64: tc2::k_pretile_w1_all<64><<<grid, 256, 0, b->stream>>>(params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    case 128: tc2::k_pretile_w1_all<128><<<grid, 256, 0, b->stream>>>(params, d.c0, d.k, d.bk, d.m, b->wtile); break;
    default: tc2::k_pretile_w1_all<192><<<grid, 256, 0, b->stream>>>(params, d.c0, d.k, d.bk, d.m, b->wtile); break;
  }
  b->launches++;
}

// 1x1 forward on the v2 engine; false when the shape is not supported (the
// caller then uses the v1 kernel).
bool tc2_conv1x1_fwd(Block* b, const LayerArgs<float>& a, int l) {
  if (a.C % 4 != 0 || !b->wtile) return false;
  const int ntiles = static_cast<int>((a.M + tc::kBM - 1) / tc::kBM);
  const uint8_t* w1t = b->wtile + b->wtile_off[l];
  auto go = [&](auto tag) -> bool {
    using Op = decltype(tag);
    const int nkb = (a.c + tc::kBK - 1) / tc::kBK;
    const size_t aux = sizeof(BnFwd) * a.c + (Op::kMmaReadsRaw ? 0 : nkb * 2 * Op::kBBytes);
    if (fixed_smem<Op>() + aux > 220 * 1024) return false;
    Op op{};
    if (!make_map_f32(&op.xmap, a.feat, a.C, a.M, a.C, 32, tc::kBM)) return false;
    op.a = a;
    op.w1t = w1t;
    launch2(b, op, ntiles, aux);
    return true;
  };
  // B resident in shared memory when all of W1's tiles fit, else streamed
  switch (tc2_bn_1x1(a.bk)) {
    case 16: return go(tc2::Fwd1x1<16, true>{}) || go(tc2::Fwd1x1<16, false>{});
    case 32: return go(tc2::Fwd1x1<32, true>{}) || go(tc2::Fwd1x1<32, false>{});
    case 48: return go(tc2::Fwd1x1<48, true>{}) || go(tc2::Fwd1x1<48, false>{});
    case 64: return go(tc2::Fwd1x1<64, true>{}) || go(tc2::Fwd1x1<64, false>{});
    case 128: return go(tc2::Fwd1x1<128, true>{}) || go(tc2::Fwd1x1<128, false>{});
    case 192: return go(tc2::Fwd1x1<192, true>{}) || go(tc2::Fwd1x1<192, false>{});
    default: return false;
  }
}

}  // namespace dpb
