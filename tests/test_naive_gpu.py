"""The Naive and SharedGradient strategy variants on the B200.

  - numerics: NaiveBlock (the unfused per-op kernels) against the oracle, with
    the fp32 contract of tests/test_block_gpu.py (forward direct, backward
    given the device's forward state);
  - the two strategies are bit-identical (same kernels in the same order;
    only where the gradient transients live differs);
  - accounting parity: the storage the variants actually hold at the end of
    the step, per arena, plus the stem / transition / head terms of the
    network around the blocks, equals predict_peak_elements (the reference's
    peak model, bit-exact through dpb_predict_peak_elements) element for
    element; the allocator's own count agrees within its rounding;
  - the memory-efficient BlockPlan arena is a fraction of the naive storage.
"""
import numpy as np
import pytest
import torch

import paper_1707_06990_b200 as P
from paper_1707_06990_b200.naive import NaiveBlock, STRATEGIES
from test_block_gpu import BWD_KEYS, _compare, oracle_backward_tf, oracle_case, to_dev

pytestmark = pytest.mark.gpu


def run_naive(s, params, x_in, acc_in, strategy):
    shp = P.BlockShape(*s)
    nb = NaiveBlock(shp, strategy)
    p = to_dev(params)
    feats = nb.forward(to_dev(x_in), p)
    z = torch.stack([sv["z"] for sv in nb.saved])
    stats = torch.cat([torch.cat([sv["ma"], sv["va"], sv["mb"], sv["vb"]]) for sv in nb.saved])
    acc = to_dev(acc_in)
    grads = torch.full((p.numel(),), float("nan"), device="cuda")
    nb.backward(p, acc, grads)
    torch.cuda.synchronize()
    return dict(feats=feats.cpu().numpy(), z=z.cpu().numpy(), stats=stats.cpu().numpy(),
                acc_out=acc.cpu().numpy(), grads=grads.cpu().numpy())


@pytest.mark.parametrize("s", [(2, 9, 7, 13, 3, 5, 20), (4, 16, 16, 24, 6, 12, 48)])
@pytest.mark.parametrize("strategy", STRATEGIES)
def test_naive_block_matches_oracle(s, strategy):
    ref = oracle_case(s, 17)
    got = run_naive(s, ref["params"], ref["x_in"], ref["acc_in"], strategy)
    bad = []
    for key in ("feats", "z", "stats"):
        _compare(bad, key, got[key], ref[key], ref["f64"][key], "fp32")
    t64 = oracle_backward_tf(s, ref["params"], got, ref["acc_in"], np.float64)
    t32 = oracle_backward_tf(s, ref["params"], got, ref["acc_in"], np.float32)
    for key in BWD_KEYS:
        assert np.all(np.isfinite(got[key])), key
        _compare(bad, key, got[key], t32[key], t64[key], "fp32")
    assert not bad, f"{strategy} {s}: " + "; ".join(bad)


def test_strategies_bit_identical():
    s = (3, 12, 10, 16, 4, 8, 32)
    ref = oracle_case(s, 3)
    a = run_naive(s, ref["params"], ref["x_in"], ref["acc_in"], "naive")
    b = run_naive(s, ref["params"], ref["x_in"], ref["acc_in"], "shared-gradient")
    for key in a:
        assert np.array_equal(a[key], b[key]), key


def _random_step(nb, shp, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    p = (torch.randn(shp.param_elems, generator=g) * 0.2 + 0.5).cuda()
    x = torch.randn((shp.n, shp.c0, shp.h, shp.w), generator=g).cuda()
    acc = torch.randn((shp.n, shp.c_out, shp.h, shp.w), generator=g).cuda()
    grads = torch.empty_like(p)
    nb.forward(x, p)
    nb.backward(p, acc, grads)
    torch.cuda.synchronize()
    return x


def _network_terms(cfg, shapes, batch, strategy):
    """The stem / transition / head terms of peak_model.hpp:56-106 (the
    network around the dense blocks): stem output, per transition its BN pool,
    conv output, pooled output (the next block's input) and two gradient
    transients, and the head's BN pool, pooled vector, logits and two
    transients.  The stem output / pooled outputs are the blocks' inputs."""
    N = batch
    total, transients = 0, []
    total += shapes[0].c0 * shapes[0].h * shapes[0].w * N                    # stem output
    for b, shp in enumerate(shapes):
        hw = shp.h * shp.w
        C = shp.c_out
        if b + 1 < len(shapes):
            tc = shapes[b + 1].c0
            total += C * hw * N                                              # bn pool
            total += tc * hw * N + tc * shapes[b + 1].h * shapes[b + 1].w * N  # conv out, pooled
            transients += [tc * hw * N, C * hw * N]
        else:
            total += C * hw * N + C * N + cfg.num_classes * N                # bn pool, GAP, logits
            transients += [C * N, C * hw * N]
    return total, transients


@pytest.mark.parametrize("blocks", [(4,), (3, 2)])
@pytest.mark.parametrize("strategy", STRATEGIES)
def test_accounting_matches_peak_model(blocks, strategy):
    if strategy == "shared-gradient" and len(blocks) > 1:
        pytest.skip("the network shares one gradient region across blocks; one block owns it here")
    cfg = P.DenseNetConfig(blocks, 8, True, 0.5, 10, 16, (3, 12, 12))
    batch = 2
    shapes = cfg.block_shapes(batch)
    pred = P.predict_peak_elements(cfg, "naive" if strategy == "naive" else "shared-grad", batch, 3, 12, 12)
    fixed, transients = _network_terms(cfg, shapes, batch, strategy)
    feature = fixed
    grad = 0
    for b, shp in enumerate(shapes):
        nb = NaiveBlock(shp, strategy)
        _random_step(nb, shp, 100 + b)
        acct = nb.accounting()
        feature += acct["cat"] + acct["bn"] + acct["owned"]
        grad += acct["grad"]
    if strategy == "naive":
        assert feature + grad + sum(transients) == pred["feature_owned"]
        assert pred["shared_grad"] == 0
    else:
        assert feature == pred["feature_owned"]
        # one block: its region (4 slots of max(transient, accumulator)) is the network's
        assert grad == pred["shared_grad"]


@pytest.mark.parametrize("strategy", STRATEGIES)
def test_device_allocation_matches_accounting(strategy):
    shp = P.BlockShape(4, 16, 16, 24, 6, 12, 48)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    nb = NaiveBlock(shp, strategy)
    x = _random_step(nb, shp, 9)
    held = torch.cuda.memory_allocated() - base
    # held also counts x, the parameters / gradients / accumulator of the
    # caller and the per-layer statistics vectors (outside the peak model)
    extra = 4 * (x.numel() + 2 * shp.param_elems + shp.n * shp.c_out * shp.h * shp.w + 4 * shp.stat_elems)
    counted = nb.retained_bytes()
    assert counted <= held <= counted + extra + 512 * 64 * shp.m


def test_efficient_arena_is_a_fraction_of_naive():
    shp = P.BlockShape(8, 16, 16, 24, 12, 12, 48)
    nb = NaiveBlock(shp, "naive")
    _random_step(nb, shp, 4)
    eff, naive_analytic = P.block_memory(shp, "fp32")
    measured = nb.retained_bytes() + 4 * shp.n * shp.c0 * shp.h * shp.w   # + the block input
    assert measured == naive_analytic
    assert eff < 0.35 * measured
