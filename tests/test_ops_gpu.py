"""Per-op device kernels (dpb_op_*) against the reference's known answers
(t/ops_test.cpp) and float64 restatements of ops.hpp."""
import numpy as np
import pytest
import torch

from conftest import rel_err
from paper_1707_06990_b200 import errors, ops

pytestmark = pytest.mark.gpu


def conv_ref(x, w, pad):
    n, cin, h, ww = x.shape
    cout, _, k, _ = w.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    oh, ow = h + 2 * pad - k + 1, ww + 2 * pad - k + 1
    out = np.zeros((n, cout, oh, ow))
    for ky in range(k):
        for kx in range(k):
            out += np.einsum("nchw,oc->nohw", xp[:, :, ky:ky + oh, kx:kx + ow], w[:, :, ky, kx])
    return out


def test_conv_identity_and_hand_sums():
    # t/ops_test.cpp:267-298
    x = torch.randn(2, 3, 4, 4, device="cuda")
    w = torch.zeros(3, 3, 1, 1, device="cuda")
    for i in range(3):
        w[i, i] = 1
    assert torch.equal(ops.conv2d_forward(x, w, 0), x)
    y = ops.conv2d_forward(torch.ones(1, 1, 3, 3, device="cuda"), torch.ones(1, 1, 3, 3, device="cuda"), 1)
    assert y[0, 0, 1, 1].item() == 9 and y[0, 0, 0, 1].item() == 6 and y[0, 0, 0, 0].item() == 4


@pytest.mark.parametrize("k,pad", [(1, 0), (3, 1)])
def test_conv_forward_backward(k, pad):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 5, 6, 7)).astype(np.float32)
    w = rng.standard_normal((4, 5, k, k)).astype(np.float32)
    y = ops.conv2d_forward(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), pad).cpu().numpy()
    assert rel_err(y, conv_ref(x.astype(np.float64), w.astype(np.float64), pad)) < 1e-5
    gy = rng.standard_normal(y.shape).astype(np.float32)
    gx, gw = ops.conv2d_backward(torch.from_numpy(gy).cuda(), torch.from_numpy(x).cuda(),
                                 torch.from_numpy(w).cuda(), pad)
    # adjoint identities: <gy, conv(x)> = <gx, x> = <gw, w>
    ip = float(np.sum(gy.astype(np.float64) * conv_ref(x.astype(np.float64), w.astype(np.float64), pad)))
    assert abs(float(np.sum(gx.cpu().numpy() * x)) - ip) / abs(ip) < 1e-4
    assert abs(float(np.sum(gw.cpu().numpy() * w)) - ip) / abs(ip) < 1e-4


def test_conv_shape_validation():
    with pytest.raises(errors.ShapeError):
        ops.conv2d_forward(torch.zeros(1, 3, 4, 4, device="cuda"), torch.zeros(2, 4, 1, 1, device="cuda"), 0)
    with pytest.raises(errors.ShapeError):
        ops.conv2d_forward(torch.zeros(1, 1, 1, 1, device="cuda"), torch.zeros(1, 1, 3, 3, device="cuda"), 0)


def test_batchnorm_statistics_and_apply():
    # t/ops_test.cpp:108-143: constant -> 0; normalised mean beta, var ~1
    x = torch.full((2, 3, 4, 4), 5.0, device="cuda")
    m, v = ops.batch_statistics(x)
    assert torch.allclose(m, torch.full_like(m, 5.0)) and torch.all(v == 0)
    g = torch.ones(3, device="cuda")
    b = torch.zeros(3, device="cuda")
    assert torch.all(ops.batchnorm_apply(x, g, b, m, v) == 0)
    x = torch.randn(4, 3, 5, 5, device="cuda") * 3 + 1
    m, v = ops.batch_statistics(x)
    xd = x.double().cpu().numpy()
    np.testing.assert_allclose(m.cpu().numpy(), xd.mean(axis=(0, 2, 3)), rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(v.cpu().numpy(), xd.var(axis=(0, 2, 3)), rtol=1e-5)
    beta = torch.tensor([0.5, -1.0, 2.0], device="cuda")
    y = ops.batchnorm_apply(x, g, beta, m, v).double().cpu().numpy()
    np.testing.assert_allclose(y.mean(axis=(0, 2, 3)), beta.cpu().numpy(), atol=1e-5)
    yr = ops.batchnorm_apply(x, g, beta, m, v, relu=True)
    assert torch.all(yr >= 0)


def test_batchnorm_backward_identities():
    # t/ops_test.cpp:202-239: dbeta = sum g; zero grad -> zero; finite difference
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 4, 5, 5))
    gam = rng.standard_normal(4) + 1
    gy = rng.standard_normal(x.shape)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    m, v = ops.batch_statistics(T(x))
    gx, dg, db = ops.batchnorm_backward(T(gy), T(x), T(gam), m, v)
    np.testing.assert_allclose(db.cpu().numpy(), gy.sum(axis=(0, 2, 3)), rtol=1e-5, atol=1e-5)

    def loss(xx):
        mu = xx.mean(axis=(0, 2, 3), keepdims=True)
        var = xx.var(axis=(0, 2, 3), keepdims=True)
        y = gam[None, :, None, None] * (xx - mu) / np.sqrt(var + 1e-5)
        return float(np.sum(y * gy))
    num = np.zeros_like(x)
    h = 1e-6
    for idx in [(0, 0, 0, 0), (1, 2, 3, 4), (2, 3, 1, 1), (0, 1, 4, 2)]:
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        num[idx] = (loss(xp) - loss(xm)) / (2 * h)
        assert abs(gx.cpu().numpy()[idx] - num[idx]) < 1e-3
    gx0, dg0, db0 = ops.batchnorm_backward(torch.zeros_like(T(x)), T(x), T(gam), m, v)
    assert torch.count_nonzero(gx0).item() == 0 and torch.count_nonzero(db0).item() == 0


def test_concat_forward_backward_order_and_errors():
    # t/ops_test.cpp:42-106: inputs land in order, channel by channel
    a = torch.randn(2, 3, 4, 5, device="cuda")
    b = torch.randn(2, 1, 4, 5, device="cuda")
    c = torch.randn(2, 4, 4, 5, device="cuda")
    out = ops.concat_forward([a, b, c])
    assert torch.equal(out, torch.cat([a, b, c], dim=1))
    parts = ops.concat_backward(out, [3, 1, 4])
    for p, ref in zip(parts, (a, b, c)):
        assert torch.equal(p, ref)
    with pytest.raises(errors.ShapeError):
        ops.concat_forward([])
    with pytest.raises(errors.ShapeError):
        ops.concat_forward([a, torch.randn(2, 1, 3, 5, device="cuda")])
    with pytest.raises(errors.ShapeError):
        ops.concat_backward(out, [3, 1, 3])


def test_relu_forward_backward_subgradient_zero():
    # t/ops_test.cpp:241-265: subgradient 0 at 0, in-place variants
    x = torch.tensor([-2.0, -0.0, 0.0, 1e-30, 3.0], device="cuda")
    y = ops.relu_forward(x)
    assert y.tolist() == [0.0, 0.0, 0.0, x[3].item(), 3.0]
    g = torch.ones_like(x)
    assert ops.relu_backward(g, x).tolist() == [0.0, 0.0, 0.0, 1.0, 1.0]
    assert ops.relu_backward(g, y).tolist() == [0.0, 0.0, 0.0, 1.0, 1.0]
    z = x.clone()
    ops.relu_forward(z, inplace=True)
    assert torch.equal(z, y)
