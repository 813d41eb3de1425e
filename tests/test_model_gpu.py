"""Whole-network training step on the GPU (dpb_model_*)
against the reference's own GraphPlan<float>::step_trace (tests/golden/model_*.npz,
oracle/gen_golden.py): same parameters (GraphPlan::build draws), same synthetic
input and labels.

Compared per parameter tensor (registration order) with the normwise relative
error ||got - ref|| / ||ref||, and the loss, against the north_star bounds:
1e-4 for the fp32 path (SIMT blocks; measured worst 4.6e-6) and 2e-2 for the
bf16 path (tcgen05 blocks and transition GEMMs; measured worst 1.6e-2).
"""
import numpy as np
import pytest
import torch

from paper_1707_06990_b200.model import DenseNetConfig, ModelPlan

pytestmark = pytest.mark.gpu

CASES = ["model_small", "model_bc", "model_k32", "model_odd"]
TOL = {"fp32": 1e-4, "bf16": 2e-2}


def _load(name):
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz"))
    return {k: g[k] for k in g.files}


def _segments(g):
    """(name, size) of every parameter tensor in registration order."""
    blocks = [int(b) for b in g["blocks"]]
    k, c0, classes = int(g["k"]), int(g["c0"]), int(g["classes"])
    in_c = int(g["in_shape"][1])
    bk = 4 * k
    segs = [("stem.w", c0 * in_c * 9)]
    c = c0
    for b, m in enumerate(blocks):
        for l in range(m):
            ci = c + l * k
            segs += [(f"b{b}.l{l}.bn_a.gamma", ci), (f"b{b}.l{l}.bn_a.beta", ci), (f"b{b}.l{l}.conv_a.w", bk * ci),
                     (f"b{b}.l{l}.bn_b.gamma", bk), (f"b{b}.l{l}.bn_b.beta", bk), (f"b{b}.l{l}.conv_b.w", k * bk * 9)]
        C = c + m * k
        if b + 1 < len(blocks):
            cout = int(np.floor(float(g["compression"]) * C))
            segs += [(f"t{b}.bn.gamma", C), (f"t{b}.bn.beta", C), (f"t{b}.conv.w", cout * C)]
            c = cout
        else:
            segs += [("head.bn.gamma", C), ("head.bn.beta", C), ("head.linear.w", classes * C),
                     ("head.linear.b", classes)]
    return segs


def _run(g, dtype):
    n, cin, h, w = (int(v) for v in g["in_shape"])
    cfg = DenseNetConfig(tuple(int(b) for b in g["blocks"]), int(g["k"]), True, float(g["compression"]),
                         int(g["classes"]), int(g["c0"]), (cin, h, w))
    plan = ModelPlan(cfg, n, dtype=dtype)
    assert plan.param_elems == g["params"].size
    params = torch.from_numpy(g["params"]).cuda()
    x = torch.from_numpy(g["x"]).cuda()
    labels = torch.from_numpy(g["labels"]).cuda()
    running = plan.initial_running()
    grads = torch.full((plan.param_elems,), float("nan"), device="cuda")
    loss = torch.zeros(1, device="cuda")
    plan.step(x, labels, params, running, grads, loss)
    plan.sync()
    out = grads.cpu().numpy(), float(loss.item()), running.cpu().numpy()
    plan.close()
    return out


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("name", CASES)
def test_model_step_matches_reference(name, dtype):
    g = _load(name)
    grads, loss, running = _run(g, dtype)
    assert np.isfinite(grads).all(), "every gradient written"
    assert abs(loss - float(g["loss"])) <= TOL[dtype] * abs(float(g["loss"]))
    o = 0
    worst = (0.0, "")
    for seg, size in _segments(g):
        ref, got = g["grads"][o:o + size].astype(np.float64), grads[o:o + size].astype(np.float64)
        err = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
        worst = max(worst, (err, seg))
        o += size
    assert o == grads.size
    assert worst[0] <= TOL[dtype], f"{name} {dtype}: worst {worst[1]} normwise error {worst[0]:.3e}"
    if dtype == "fp32":
        # and elementwise with the reference's own measure, rel_err(a, b) =
        # |a - b| / max(1, |a|, |b|) (gradcheck.hpp:14-17), at its 1e-4 contract
        ref = g["grads"].astype(np.float64)
        got = grads.astype(np.float64)
        rel = np.abs(got - ref) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(ref)))
        assert rel.max() <= 1e-4, f"{name}: elementwise rel_err {rel.max():.3e} at {int(rel.argmax())}"


def test_model_step_is_deterministic():
    g = _load("model_bc")
    a, la, _ = _run(g, "bf16")
    b, lb, _ = _run(g, "bf16")
    assert la == lb
    np.testing.assert_array_equal(a, b)


def test_model_bad_label_raises():
    from paper_1707_06990_b200.errors import LabelError
    g = _load("model_small")
    n, cin, h, w = (int(v) for v in g["in_shape"])
    cfg = DenseNetConfig(tuple(int(b) for b in g["blocks"]), int(g["k"]), True, float(g["compression"]),
                         int(g["classes"]), int(g["c0"]), (cin, h, w))
    plan = ModelPlan(cfg, n)
    params = torch.from_numpy(g["params"]).cuda()
    x = torch.from_numpy(g["x"]).cuda()
    labels = torch.full((n,), 99, dtype=torch.int32, device="cuda")
    grads = torch.zeros(plan.param_elems, device="cuda")
    loss = torch.zeros(1, device="cuda")
    plan.step(x, labels, params, plan.initial_running(), grads, loss)
    with pytest.raises(LabelError):
        plan.sync()
    plan.close()


def test_model_graph_replay_matches_eager():
    """dpb_model_step on a created stream captures the step into a CUDA graph and
    replays it while the buffers stay the same, re-capturing when they change:
    bit-identical to the eager launches (DPB_MODEL_NO_GRAPH semantics: a default
    stream launches eagerly)."""
    g = _load("model_bc")
    n, cin, h, w = (int(v) for v in g["in_shape"])
    cfg = DenseNetConfig(tuple(int(b) for b in g["blocks"]), int(g["k"]), True, float(g["compression"]),
                         int(g["classes"]), int(g["c0"]), (cin, h, w))
    params = torch.from_numpy(g["params"]).cuda()
    x = torch.from_numpy(g["x"]).cuda()
    labels = torch.from_numpy(g["labels"]).cuda()

    def run(stream):
        plan = ModelPlan(cfg, n, dtype="bf16", stream=stream)
        running = plan.initial_running()
        loss = torch.zeros(1, device="cuda")
        grads = torch.empty(plan.param_elems, device="cuda")
        outs = []
        for step in range(4):
            if step == 2:  # new buffers: the graph is captured again
                grads = torch.empty(plan.param_elems, device="cuda")
            grads.fill_(float("nan"))
            torch.cuda.synchronize()
            plan.step(x, labels, params, running, grads, loss)
            plan.sync()
            torch.cuda.synchronize()
            outs.append((grads.cpu().numpy().copy(), loss.cpu().numpy().copy(), running.cpu().numpy().copy()))
        plan.close()
        return outs

    eager = run(None)
    graphed = run(torch.cuda.Stream())
    for step, (a, b) in enumerate(zip(eager, graphed)):
        for t_a, t_b, what in zip(a, b, ("grads", "loss", "running")):
            assert np.isfinite(t_b).all(), f"step {step} {what}"
            assert np.array_equal(t_a, t_b), f"step {step} {what} differs between graph replay and eager"


@pytest.mark.parametrize("stem", ["3x3", "imagenet"])
def test_model_input_refill_overlapped_with_the_step(stem):
    """dpb_model_wait_input: the next batch copied into the same input buffers on
    another stream once the previous step has read them (the tensor-core
    ImageNet stem releases them after the forward's loss, the 3x3 stem after the
    whole step) gives the same losses and gradients, bit for bit, as copying
    between fully synchronised steps."""
    n = 4
    in_shape = (3, 32, 32) if stem == "imagenet" else (3, 16, 16)
    cfg = DenseNetConfig((2, 2), 8, True, 0.5, 10, 16, in_shape, stem=stem)
    gen = torch.Generator().manual_seed(3)
    xa = torch.randn(n, *in_shape, generator=gen).cuda()
    xb = torch.randn(n, *in_shape, generator=gen).cuda()
    labels = (torch.arange(n, dtype=torch.int32) % 10).cuda()
    s, cs = torch.cuda.Stream(), torch.cuda.Stream()

    def run(overlap):
        plan = ModelPlan(cfg, n, dtype="bf16", stream=s)
        params = plan.init_params(seed=5)
        running = plan.initial_running()
        grads = torch.empty(plan.param_elems, device="cuda")
        loss = torch.zeros(1, device="cuda")
        x = xa.clone()
        torch.cuda.synchronize()
        plan.step(x, labels, params, running, grads, loss)
        with torch.cuda.stream(s):
            g1, l1 = grads.clone(), loss.clone()
        if overlap:
            plan.wait_input(cs)
            with torch.cuda.stream(cs):
                x.copy_(xb)
                ev = torch.cuda.Event()
                ev.record(cs)
            s.wait_event(ev)
        else:
            torch.cuda.synchronize()
            x.copy_(xb)
            torch.cuda.synchronize()
        plan.step(x, labels, params, running, grads, loss)
        plan.sync()
        torch.cuda.synchronize()
        out = [t.cpu().numpy() for t in (g1, l1, grads, loss, running)]
        plan.close()
        return out

    for a, b in zip(run(False), run(True)):
        np.testing.assert_array_equal(a, b)
