"""Dense-block parity on the B200: libdpb.so (through the C ABI) against the
oracle restatement and the reference's own golden vectors.

Parity contract (BASELINE.json north_star tolerances):
  forward  (features, bottleneck outputs, batch statistics, running
           statistics): compared with the reference directly;
  backward (block-gradient accumulator, every parameter gradient): compared
           with the reference's backward GIVEN THE SAME FORWARD STATE (the
           device's stored features / z / statistics fed to the oracle).  A
           ReLU mask evaluated on a pre-activation within one fp32 rounding
           of zero can legitimately differ between any two fp32 evaluations
           (the reference's own f32 and f64 runs differ that way) and moves
           one pixel's gradient by O(1); with the forward state shared, the
           device evaluates the mask with the reference's exact float
           expression (dpb_common.cuh relu_mask_ref) and the comparison is
           free of that effect.
  fp32 path: rel_err = |a-b| / max(1, |a|, |b|) <= 1e-4 elementwise (the
           reference's own metric, dp/gradcheck.hpp:14-17) against the
           reference in float64; against the reference in float32 the bound
           is max(1e-4, 2 x that run's own deviation from float64), because
           the reference's sequential fp32 sums are themselves off by up to
           ~2e-4 on cancelling gradient sums.
  bf16 path: ||a-b||_2 / ||b||_2 <= 2e-2 per tensor against float64.
"""
import numpy as np
import pytest
import torch

from conftest import GOLDEN_CASES, load_golden, norm_err, rel_err
import paper_1707_06990_b200 as P
from paper_1707_06990_b200 import errors
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_TOL = 2e-2


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def nchw_to_nhwc(a):
    return np.ascontiguousarray(np.moveaxis(np.asarray(a), 1, -1))


def nhwc_to_nchw(a):
    return np.ascontiguousarray(np.moveaxis(np.asarray(a), -1, 1))


def run_device(s, params, x_in, running_in, acc_in, dtype, layout="nchw"):
    plan = P.BlockPlan(P.BlockShape(*s), dtype=dtype, layout=layout)
    p = to_dev(params)
    run = to_dev(running_in)
    x = to_dev(x_in if layout == "nchw" else nchw_to_nhwc(x_in))
    plan.forward(x, p, run, True)
    feats, z, stats = plan.feats(), plan.z(), plan.stats()
    acc = to_dev(acc_in if layout == "nchw" else nchw_to_nhwc(acc_in))
    grads = torch.full((p.numel(),), float("nan"), device="cuda")
    plan.backward(p, acc, grads)
    plan.sync()
    acc_np = acc.cpu().numpy()
    if layout == "nhwc":
        acc_np = nhwc_to_nchw(acc_np)
    out = dict(feats=feats.cpu().numpy(), z=z.cpu().numpy(), stats=stats.cpu().numpy(),
               running=run.cpu().numpy(), acc_out=acc_np, grads=grads.cpu().numpy())
    plan.close()
    return out


def oracle_run(s, params, x, acc, run0, dt):
    shp = O.BlockShape(*s)
    feats, z, stats, run = O.block_forward(shp, params.astype(dt), x.astype(dt), run0.astype(dt), True)
    acc_out, grads = O.block_backward(shp, params.astype(dt), feats, z, stats, acc.astype(dt))
    return dict(feats=feats, z=z, stats=stats, running=run, acc_out=acc_out, grads=grads)


def oracle_backward_tf(s, params, got, acc, dt):
    """The reference backward fed the device's forward state (teacher forced)."""
    shp = O.BlockShape(*s)
    acc_out, grads = O.block_backward(shp, params.astype(dt), got["feats"].astype(dt),
                                      got["z"].astype(dt), got["stats"].astype(dt), acc.astype(dt))
    return dict(acc_out=acc_out, grads=grads)


def oracle_case(s, seed, perturb=True):
    shp = O.BlockShape(*s)
    params = O.random_block_params(shp, seed, np.float32, perturb_bn=perturb)
    x = O.rng_normal(seed + 99, shp.n * shp.c0 * shp.h * shp.w, np.float32).reshape(shp.n, shp.c0, shp.h, shp.w)
    acc = O.rng_normal(seed + 100, shp.n * shp.c_out * shp.h * shp.w, np.float32).reshape(
        shp.n, shp.c_out, shp.h, shp.w)
    run0 = shp.initial_running(np.float32)
    ref = dict(params=params, x_in=x, acc_in=acc, running_in=run0)
    ref.update(oracle_run(s, params, x, acc, run0, np.float32))
    ref["f64"] = oracle_run(s, params, x, acc, run0, np.float64)
    return ref


FWD_KEYS = ("feats", "z", "stats", "running")
BWD_KEYS = ("acc_out", "grads")


def _compare(bad, key, got, r32, r64, dtype):
    if dtype == "fp32":
        e64 = rel_err(got, r64)
        if r32 is None:
            if not e64 <= FP32_TOL:
                bad.append(f"{key}: rel_err vs f64 {e64:.3e}")
            return
        own = rel_err(r32, r64)
        e32 = rel_err(got, r32)
        if not (e64 <= FP32_TOL or e32 <= max(FP32_TOL, 2 * own)):
            bad.append(f"{key}: rel_err vs f64 {e64:.3e}, vs f32 {e32:.3e} (reference f32 own error {own:.3e})")
    else:
        e = norm_err(got, r64)
        if not e <= BF16_TOL:
            bad.append(f"{key}: norm_err {e:.3e}")


def check(got, ref, dtype, label="", s=None):
    """ref: the reference run (float32 or float64) on the case inputs, with
    ref['f64'] the float64 run when ref is float32."""
    bad = []
    is64 = ref["grads"].dtype == np.float64
    r64 = ref if is64 else ref["f64"]
    r32 = None if is64 else ref
    for key in FWD_KEYS + BWD_KEYS:
        assert np.all(np.isfinite(got[key])), f"{label} {key} has non-finite values"
    for key in FWD_KEYS:
        _compare(bad, key, got[key], None if r32 is None else r32[key], r64[key], dtype)
    # backward given the device's forward state
    shape = s if s is not None else tuple(int(v) for v in ref["shape"])
    t64 = oracle_backward_tf(shape, ref["params"], got, ref["acc_in"], np.float64)
    t32 = None if is64 else oracle_backward_tf(shape, ref["params"], got, ref["acc_in"], np.float32)
    for key in BWD_KEYS:
        _compare(bad, key, got[key], None if t32 is None else t32[key], t64[key], dtype)
    assert not bad, f"{label} {dtype}: " + "; ".join(bad)


@pytest.mark.parametrize("name", GOLDEN_CASES)
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_block_matches_reference_golden(name, dtype):
    g = load_golden(name)
    if g["params"].dtype == np.float32:
        # the same inputs through the reference arithmetic in float64
        g["f64"] = oracle_run(g["shape_tuple"], g["params"], g["x_in"], g["acc_in"], g["running_in"],
                              np.float64)
    got = run_device(g["shape_tuple"], g["params"], g["x_in"], g["running_in"], g["acc_in"], dtype)
    check(got, g, dtype, name, g["shape_tuple"])


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
def test_block_matches_oracle_medium(dtype, layout):
    # cfg1 channel geometry (c0=24, k=12, bk=48), 6 layers, 4x16x16
    s = (4, 16, 16, 24, 6, 12, 48)
    ref = oracle_case(s, 21)
    got = run_device(s, ref["params"], ref["x_in"], ref["running_in"], ref["acc_in"], dtype, layout)
    check(got, ref, dtype, f"medium-{layout}", s)


@pytest.mark.parametrize("s", [
    (2, 9, 7, 13, 3, 5, 20),     # ragged channels, odd field, bk not a multiple of 16
    (3, 14, 14, 40, 2, 32, 128), # k=32 geometry (DenseNet-121/264-k32), bk=128 > 64 (N tiling)
    (1, 7, 7, 96, 2, 48, 192),   # k=48 geometry (DenseNet-264-k48), 7x7 field, batch 1
    # wide inputs at 7x7 (DenseNet-264 block 4): W1 streamed per K block, and so
    # few pixel tiles that the 1x1 forward splits its 192 columns across CTAs
    (2, 7, 7, 520, 2, 48, 192),
    (16, 7, 7, 1728, 1, 48, 192),
    # the real widths of DenseNet-264: block 3's widest layer (c = 3,408), block
    # 4's (c = 3,936 + 48) at k = 48 / bk = 192 (Dgrad1x1<128, 4>: 32 column
    # tiles), and k = 32 / bk = 128 blocks 3-4 (c0 >= 512: 256-column dgrad tiles)
    (2, 14, 14, 3408, 1, 48, 192),
    (4, 7, 7, 3936, 1, 48, 192),
    (4, 14, 14, 2240, 1, 32, 128),
    (8, 7, 7, 1120, 2, 32, 128),
    # 56x56 with more halo tiles than SMs: the 3x3 forward picks K chunks for
    # two CTAs per SM — with the two-slot raw ring at k = 32, the one-slot
    # ring at k = 48 (bk = 192)
    (8, 56, 56, 64, 1, 32, 128),
    (8, 56, 56, 64, 1, 48, 192),
])
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_block_matches_oracle_shapes(s, dtype):
    ref = oracle_case(s, 5)
    got = run_device(s, ref["params"], ref["x_in"], ref["running_in"], ref["acc_in"], dtype)
    check(got, ref, dtype, str(s), s)


@pytest.fixture(scope="module")
def cfg1_ref():
    # BASELINE config 1 at full size: 16x32x32, c0=24, k=12, m=12 (oracle ~20 s)
    return oracle_case((16, 32, 32, 24, 12, 12, 48), 7)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_block_matches_oracle_cfg1_full(cfg1_ref, dtype):
    s = (16, 32, 32, 24, 12, 12, 48)
    got = run_device(s, cfg1_ref["params"], cfg1_ref["x_in"], cfg1_ref["running_in"], cfg1_ref["acc_in"],
                     dtype)
    check(got, cfg1_ref, dtype, "cfg1", s)


def _random_plan_inputs(s, seed, layout="nhwc"):
    shp = P.BlockShape(*s)
    g = torch.Generator(device="cpu").manual_seed(seed)
    params = torch.randn(shp.param_elems, generator=g) * 0.2
    for l, o in enumerate(shp.param_offsets()):
        c = shp.c_in(l)
        params[o:o + c] += 1.0                      # gamma_a around 1
        gb = o + 2 * c + shp.bk * c
        params[gb:gb + shp.bk] += 1.0               # gamma_b around 1
    x = torch.randn((shp.n, shp.h, shp.w, shp.c0) if layout == "nhwc" else (shp.n, shp.c0, shp.h, shp.w),
                    generator=g)
    return shp, params.cuda(), x.cuda()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_backward_is_linear_in_upstream_gradient(dtype):
    # For a fixed forward, the block backward is linear in grad_acc: a
    # size-independent property checked at a DenseNet-264-k48 block-3 shape.
    s = (2, 14, 14, 384, 4, 48, 192)
    shp, p, x = _random_plan_inputs(s, 3)
    plan = P.BlockPlan(shp, dtype=dtype, layout="nhwc")
    run = shp.initial_running()
    plan.forward(x, p, run, False)
    M = shp.pixels
    g1 = torch.randn(M, shp.c_out, device="cuda")
    g2 = torch.randn(M, shp.c_out, device="cuda")
    outs = []
    for g in (g1, g2, 2.0 * g1 - 3.0 * g2):
        acc = g.clone()
        gr = torch.empty(shp.param_elems, device="cuda")
        plan.backward(p, acc, gr)
        outs.append((acc, gr))
    plan.sync()
    for i in (0, 1):
        lhs = outs[2][i].double()
        rhs = 2.0 * outs[0][i].double() - 3.0 * outs[1][i].double()
        err = (lhs - rhs).norm() / rhs.norm()
        # bf16: the tensor-core backward rounds its GEMM operands to bf16
        assert err < (1e-5 if dtype == "fp32" else 1e-2), err


def test_zero_upstream_gives_zero_gradients():
    # t/graph_test.cpp:164-185
    s = (2, 8, 8, 16, 3, 8, 32)
    shp, p, x = _random_plan_inputs(s, 4)
    plan = P.BlockPlan(shp, dtype="fp32", layout="nhwc")
    plan.forward(x, p, shp.initial_running(), True)
    acc = torch.zeros(shp.pixels, shp.c_out, device="cuda")
    gr = torch.full((shp.param_elems,), 7.0, device="cuda")
    plan.backward(p, acc, gr)
    plan.sync()
    assert torch.count_nonzero(gr).item() == 0
    assert torch.count_nonzero(acc).item() == 0


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_deterministic_bitwise_rerun(dtype):
    # fixed-order reductions: two runs produce identical bits (graph_test 134-141)
    s = (8, 16, 16, 24, 4, 12, 48)
    shp, p, x = _random_plan_inputs(s, 5)
    res = []
    for _ in range(2):
        plan = P.BlockPlan(shp, dtype=dtype, layout="nhwc")
        run = shp.initial_running()
        plan.forward(x, p, run, True)
        acc = torch.ones(shp.pixels, shp.c_out, device="cuda")
        gr = torch.empty(shp.param_elems, device="cuda")
        plan.backward(p, acc, gr)
        plan.sync()
        res.append((plan.feats(), acc, gr, run))
    for a, b in zip(*res):
        assert torch.equal(a, b)


def test_eval_with_batch_stats_equals_train():
    # ops.hpp:196-199: eval normalises with running stats; feeding the batch
    # statistics as the running statistics must reproduce the train forward.
    s = (4, 8, 8, 16, 3, 8, 32)
    shp, p, x = _random_plan_inputs(s, 6)
    plan = P.BlockPlan(shp, dtype="fp32", layout="nhwc")
    plan.forward(x, p, shp.initial_running(), True)
    train_feats = plan.feats()
    stats = plan.stats()
    plan.forward_eval(x, p, stats)
    plan.sync()
    assert torch.equal(plan.feats(), train_feats)


def test_errors_map_to_reference_classes():
    shp = P.BlockShape(1, 1, 1, 4, 1, 2, 8)
    plan = P.BlockPlan(shp, dtype="fp32", layout="nchw")
    p = torch.zeros(shp.param_elems, device="cuda")
    with pytest.raises(errors.DegenerateBatchError):
        plan.forward(torch.zeros(1, 4, 1, 1, device="cuda"), p, shp.initial_running(), True)
    shp2 = P.BlockShape(2, 2, 2, 4, 1, 2, 8)
    plan2 = P.BlockPlan(shp2, dtype="fp32")
    with pytest.raises(errors.ProtocolError):
        plan2.backward(torch.zeros(shp2.param_elems, device="cuda"),
                       torch.zeros(2, shp2.c_out, 2, 2, device="cuda"),
                       torch.zeros(shp2.param_elems, device="cuda"))
