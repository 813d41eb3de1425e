"""Whole-network training steps on the GPU (dpb_model_step) against the
reference's public GraphPlan forward / compute_loss / backward, including BN
running statistics and the ImageNet stem
(tests/golden/train_*.npz, oracle/gen_golden.py TRAIN_CASES):

* train_small / train_bc100_b64 — the reference network (3x3 stem), BC-100 at
  its bench shape (BASELINE configs[1]);
* train_imagenet_* — the ImageNet stem (7x7/2 conv, BN, ReLU, 3x3/2 max-pool)
  composed from the reference's ops (ref_driver.cpp);
* train_d264k{32,48}_56 — DenseNet-264 (BASELINE configs[3]/[4]) in the
  reference's own 56x56 geometry, batch 2; train_d264k32_224 — the bench
  headline network with the ImageNet stem at 224x224, batch 2.  These are
  compared through per-tensor sketches (oracle.sketch: random projections
  give an unbiased normwise-error estimate; sampled elements give rel_err).

Parameters: GraphPlan::build's for the case seed (init_params, bit-identical:
tests/test_model_host.py); input Rng(seed + 99); labels i % classes.
Tolerances (north_star): fp32 path 1e-4, bf16 tensor-core path 2e-2, per
tensor normwise; elementwise rel_err (dp/gradcheck.hpp:14-17) <= 1e-4 on the
fp32 path for the fully stored cases.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1707_06990_b200.model import DenseNetConfig, ModelPlan, init_params
from conftest import rel_err

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"fp32": 1e-4, "bf16": 2e-2}
SMALL = ["train_small", "train_imagenet_small", "train_imagenet_k32", "train_bc100_b64"]
LARGE = ["train_d264k32_56", "train_d264k48_56", "train_d264k32_224"]


def _load(name):
    path = os.path.join(GOLD, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} fixture not generated")
    return dict(np.load(path))


def _meta(g):
    n, c, h, w = (int(v) for v in g["in_shape"])
    stem = int(g["stem"])
    cfg = DenseNetConfig(tuple(int(b) for b in g["blocks"]), int(g["k"]), True, float(g["compression"]),
                         int(g["classes"]), int(g["c0"]), (c, h, w), stem="imagenet" if stem else "3x3")
    return cfg, n, stem


def _run(g, dtype):
    cfg, n, stem = _meta(g)
    seed = int(g["seed"])
    plan = ModelPlan(cfg, n, dtype=dtype)
    params = torch.from_numpy(init_params(cfg, seed)).cuda()
    x = torch.from_numpy(O.rng_normal(seed + 99, n * int(np.prod(cfg.in_shape)), np.float32)).cuda()
    labels = (torch.arange(n, dtype=torch.int32) % cfg.num_classes).cuda()
    running = plan.initial_running()
    grads = torch.full((plan.param_elems,), float("nan"), device="cuda")
    loss = torch.zeros(1, device="cuda")
    plan.step(x, labels, params, running, grads, loss)
    plan.sync()
    out = grads.cpu().numpy(), float(loss.item()), running.cpu().numpy()
    plan.close()
    return out


def _segs(g):
    cfg, _, stem = _meta(g)
    return (O.model_segments(cfg.block_sizes, cfg.growth_rate, cfg.compression, cfg.num_classes, cfg.c0,
                             cfg.in_shape[0], stem),
            O.running_segments(cfg.block_sizes, cfg.growth_rate, cfg.compression, cfg.c0, stem))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("name", SMALL)
def test_train_step_matches_reference(name, dtype):
    g = _load(name)
    grads, loss, running = _run(g, dtype)
    gsegs, rsegs = _segs(g)
    assert np.isfinite(grads).all() and np.isfinite(running).all()
    assert abs(loss - float(g["loss"])) <= TOL[dtype] * abs(float(g["loss"]))
    for what, got, ref, segs in (("grads", grads, g["grads"], gsegs), ("running", running, g["running"], rsegs)):
        o, worst = 0, (0.0, "")
        for seg, size in segs:
            a, b = got[o:o + size].astype(np.float64), ref[o:o + size].astype(np.float64)
            err = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
            worst = max(worst, (err, seg))
            if dtype == "fp32":
                assert rel_err(a, b) <= 1e-4, f"{name} {what} {seg}: elementwise rel_err {rel_err(a, b):.3e}"
            o += size
        assert o == got.size
        assert worst[0] <= TOL[dtype], f"{name} {dtype} {what}: worst {worst[1]} normwise {worst[0]:.3e}"


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("name", LARGE)
def test_train_step_matches_reference_at_scale(name, dtype):
    g = _load(name)
    grads, loss, running = _run(g, dtype)
    gsegs, rsegs = _segs(g)
    assert np.isfinite(grads).all() and np.isfinite(running).all()
    assert abs(loss - float(g["loss"])) <= TOL[dtype] * abs(float(g["loss"]))
    for what, got, segs in (("grads", grads, gsegs), ("running", running, rsegs)):
        ref = {k[len(what) + 1:]: v for k, v in g.items() if k.startswith(what + "_")}
        est, rel = O.sketch_errors(got, ref, segs)
        i = int(np.argmax(est))
        assert est[i] <= TOL[dtype], f"{name} {dtype} {what}: {segs[i][0]} normwise estimate {est[i]:.3e}"
        if dtype == "fp32":
            assert rel.max() <= 1e-4, f"{name} {what}: sampled elementwise rel_err {rel.max():.3e}"
