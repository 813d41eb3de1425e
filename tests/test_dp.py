"""Data-parallel host logic on CPU: world size 2 over gloo.

Parity for P > 1: run the oracle once per shard with identical
parameters, average the gradients in float64 on the host, and compare with what
`GradientBuckets` produces from the per-rank gradients (per-block async buckets
and the one-shot path). No GPU: the device backward is replaced by the oracle
here; tests/test_block_gpu.py covers the device backward itself.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1707_06990_b200.dp import GradientBuckets, shard_range

# two dense blocks of different geometry -> two buckets
SHAPES = [(4, 5, 5, 6, 3, 4, 8), (4, 3, 3, 9, 2, 5, 12)]
WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(shape, seed):
    s = O.BlockShape(*shape)
    params = O.random_block_params(s, seed, np.float64)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((s.n, s.c0, s.h, s.w))
    acc = rng.standard_normal((s.n, s.c_out, s.h, s.w))
    return s, params, x, acc


def _shard_grads(shape, seed, lo, hi):
    s, params, x, acc = _inputs(shape, seed)
    ss = O.BlockShape(hi - lo, *shape[1:])
    feats, z, stats, run = O.block_forward(ss, params, x[lo:hi], None, True)
    _, grads = O.block_backward(ss, params, feats, z, stats, acc[lo:hi])
    return grads, run


def _worker(rank, port, mode, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        buckets = GradientBuckets([O.BlockShape(*s).param_size for s in SHAPES])
        for i, shape in enumerate(SHAPES):
            lo, hi = shard_range(shape[0], rank, WORLD)
            g, run = _shard_grads(shape, 10 + i, lo, hi)
            buckets.view(i).copy_(torch.from_numpy(g.astype(np.float32)))
            np.save(os.path.join(out_dir, f"run_{rank}_{i}.npy"), run)
        if mode == "bucketed":
            for i in reversed(range(len(SHAPES))):   # backward completes blocks in reverse
                buckets.reduce_block(i)
            flat = buckets.finish()
        else:
            flat = buckets.reduce_all()
        np.save(os.path.join(out_dir, f"flat_{rank}.npy"), flat.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["bucketed", "oneshot"])
def test_gloo_ws2_gradient_average_matches_per_shard_oracle(tmp_path, mode):
    mp.spawn(_worker, args=(_free_port(), mode, str(tmp_path)), nprocs=WORLD, join=True)
    expect = []
    for i, shape in enumerate(SHAPES):
        per_rank = [_shard_grads(shape, 10 + i, *shard_range(shape[0], r, WORLD))[0] for r in range(WORLD)]
        expect.append(np.mean(per_rank, axis=0))
    expect = np.concatenate(expect)
    flats = [np.load(tmp_path / f"flat_{r}.npy") for r in range(WORLD)]
    # every rank holds the same averaged gradient, equal to the fp64 host average
    np.testing.assert_array_equal(flats[0], flats[1])
    assert np.max(np.abs(flats[0] - expect)) <= 1e-6 * max(1.0, np.max(np.abs(expect)))
    # BN running statistics stay per rank: rank r's equal shard r's oracle run
    for r in range(WORLD):
        for i, shape in enumerate(SHAPES):
            _, run = _shard_grads(shape, 10 + i, *shard_range(shape[0], r, WORLD))
            np.testing.assert_array_equal(np.load(tmp_path / f"run_{r}_{i}.npy"), run)
    # per-GPU BN: the shard average is NOT the full-batch gradient (the reference semantics)
    s, params, x, acc = _inputs(SHAPES[0], 10)
    feats, z, stats, _ = O.block_forward(s, params, x, None, True)
    _, full = O.block_backward(s, params, feats, z, stats, acc)
    assert np.max(np.abs(full - expect[:full.size])) > 1e-6


def test_shard_range():
    assert [shard_range(128, r, 2) for r in range(2)] == [(0, 64), (64, 128)]
    assert shard_range(64, 0, 1) == (0, 64)
    with pytest.raises(ValueError):
        shard_range(65, 0, 2)
    with pytest.raises(ValueError):
        shard_range(1, 0, 2)
    with pytest.raises(ValueError):
        shard_range(64, 2, 2)


def test_buckets_single_process_views_and_identity():
    b = GradientBuckets([3, 5, 2])
    assert b.flat.numel() == 10
    b.view(1).fill_(2.0)
    assert b.flat[3:8].eq(2.0).all() and b.flat[:3].eq(0).all()
    # world 1 (no process group): reductions are the identity
    assert torch.equal(b.reduce_all(), b.flat)
    b.reduce_block(0)
    assert torch.equal(b.finish(), b.flat)
    with pytest.raises(ValueError):
        GradientBuckets([3, 0])


# ---- the whole-network bucket schedule of dpb_model_step (gloo, world size 2) ----
NET = dict(blocks=(2, 2), k=4, compression=0.5, classes=10, c0=8, shape=(8, 3, 8, 8), seed=21)


def _net_cfg():
    from paper_1707_06990_b200.model import DenseNetConfig
    n, c, h, w = NET["shape"]
    return DenseNetConfig(NET["blocks"], NET["k"], True, NET["compression"], NET["classes"], NET["c0"], (c, h, w))


def _net_shard_grads(lo, hi):
    """The reference's training step on images [lo, hi) of the global batch."""
    from paper_1707_06990_b200.model import init_params
    n, c, h, w = NET["shape"]
    x = O.rng_normal(NET["seed"] + 99, n * c * h * w, np.float32).reshape(n, c, h, w)
    p = init_params(_net_cfg(), NET["seed"])
    _, g, run = O.ref_model_train_step(NET["blocks"], NET["k"], NET["compression"], NET["classes"], NET["c0"],
                                       (hi - lo, c, h, w), NET["seed"], 0, p, x[lo:hi])
    return g, run


def _net_worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_1707_06990_b200.dp import model_buckets
        g, run = _net_shard_grads(*shard_range(NET["shape"][0], rank, WORLD))
        flat = torch.from_numpy(g.copy())
        for begin, end in model_buckets(_net_cfg()):   # dpb_model_step's issue order
            v = flat[begin:end]
            dist.all_reduce(v)
            v.mul_(1.0 / WORLD)
        np.save(os.path.join(out_dir, f"net_{rank}.npy"), flat.numpy())
        np.save(os.path.join(out_dir, f"netrun_{rank}.npy"), run)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not os.path.exists(O.REF_SO), reason="oracle/_ref not built (needs /root/reference)")
def test_gloo_ws2_model_bucket_schedule_matches_host_average(tmp_path):
    """Per-rank reference gradients of the whole network reduced bucket by bucket in
    dpb_model_step's order equal the fp64 host average of the per-shard steps, and
    the buckets cover every parameter exactly once (per-GPU BN: running stats stay
    per rank)."""
    from paper_1707_06990_b200.dp import model_buckets
    from paper_1707_06990_b200.model import model_sizes
    b = model_buckets(_net_cfg())
    assert sorted(b)[0][0] == 0 and sorted(b)[-1][1] == model_sizes(_net_cfg())[0]
    assert all(x[1] == y[0] for x, y in zip(sorted(b), sorted(b)[1:]))
    mp.spawn(_net_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    shards = [_net_shard_grads(*shard_range(NET["shape"][0], r, WORLD)) for r in range(WORLD)]
    expect = np.mean([g.astype(np.float64) for g, _ in shards], axis=0)
    flats = [np.load(tmp_path / f"net_{r}.npy") for r in range(WORLD)]
    np.testing.assert_array_equal(flats[0], flats[1])
    assert np.max(np.abs(flats[0] - expect)) <= 1e-6 * max(1.0, np.max(np.abs(expect)))
    for r in range(WORLD):
        np.testing.assert_array_equal(np.load(tmp_path / f"netrun_{r}.npy"), shards[r][1])
