"""tcgen05 engine self-test: plain GEMM through dpb_selftest_tc_gemm for every
operand major, both precisions (bf16, bf16x3 split) and the N tiles the
dense-block ops use; plus the per-CTA column sums of the epilogue."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_1707_06990_b200._lib import check, lib

pytestmark = pytest.mark.gpu


def tc_gemm(A, B, M, N, K, bn, a_mn, b_mn, split):
    D = torch.full((M, N), float("nan"), device="cuda")
    cs = torch.zeros(((M + 127) // 128, N, 2), device="cuda")
    Ad = (A.t().contiguous() if a_mn else A).cuda()
    Bd = (B.t().contiguous() if b_mn else B).cuda()
    check(lib().dpb_selftest_tc_gemm(C.c_void_p(Ad.data_ptr()), C.c_void_p(Bd.data_ptr()),
                                     C.c_void_p(D.data_ptr()), C.c_void_p(cs.data_ptr()), M, N, K, bn,
                                     a_mn, b_mn, split, None))
    torch.cuda.synchronize()
    return D.cpu().double(), cs.cpu().double()


@pytest.mark.parametrize("M,N,K,bn", [(128, 16, 64, 16), (300, 48, 200, 48), (256, 64, 96, 64),
                                      (384, 192, 160, 192), (200, 100, 72, 128)])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("split", [0, 1])
def test_tc_gemm(M, N, K, bn, a_mn, b_mn, split):
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K + 17 * a_mn + 5 * b_mn + split)
    A = torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g)
    D, cs = tc_gemm(A, B, M, N, K, bn, a_mn, b_mn, split)
    exact = A.double() @ B.double().t()
    if split:
        ref, tol = exact, 2e-5
    else:
        ref, tol = A.bfloat16().double() @ B.bfloat16().double().t(), 1e-5
    err = (D - ref).norm() / ref.norm()
    assert torch.isfinite(D).all()
    assert err < tol, f"normwise error {err:.3e}"
    # per-CTA column sums (sum, sum of squares) of the epilogue
    for cta in range(cs.shape[0]):
        rows = D[cta * 128:(cta + 1) * 128]
        np.testing.assert_allclose(cs[cta, :, 0].numpy(), rows.sum(0).numpy(), rtol=1e-4, atol=1e-3)
        np.testing.assert_allclose(cs[cta, :, 1].numpy(), (rows ** 2).sum(0).numpy(), rtol=1e-4, atol=1e-3)
