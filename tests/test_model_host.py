"""Host-side model arithmetic against the reference (CPU, no GPU needed).

* dpb_model_init_params replays GraphPlan<T>::build's Rng draws bit for bit
  (graph.hpp:351-390, :405-600; rng.hpp:36-49): compared with the reference's
  own params() in the committed model goldens and, when oracle/_ref is built,
  at DenseNet-264 scale.
* the ImageNet stem's layout: parameter / running-statistics counts.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1707_06990_b200.model import CONFIGS, DenseNetConfig, init_params, model_sizes

GOLD = os.path.join(os.path.dirname(__file__), "golden")
HAVE_REF = os.path.exists(O.REF_SO)


def _cfg(g, stem="3x3"):
    n, c, h, w = (int(v) for v in g["in_shape"])
    return DenseNetConfig(tuple(int(b) for b in g["blocks"]), int(g["k"]), True, float(g["compression"]),
                          int(g["classes"]), int(g["c0"]), (c, h, w), stem=stem)


@pytest.mark.parametrize("name", ["model_small", "model_bc", "model_k32", "model_odd"])
def test_init_params_equal_reference_params_bitwise(name):
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    p = init_params(_cfg(g), int(g["seed"]))
    assert p.dtype == np.float32 and p.size == g["params"].size
    assert np.array_equal(p.view(np.uint32), g["params"].view(np.uint32))


@pytest.mark.parametrize("name", ["d264k32@56", "d264k48@56"])
def test_init_params_d264_sha_matches_reference(name):
    kats = json.load(open(os.path.join(GOLD, "kats.json")))
    p = init_params(CONFIGS[name], 7)
    assert hashlib.sha256(p.tobytes()).hexdigest() == kats["params_sha256_seed7"][name]


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")
def test_init_params_d264k48_equal_reference_live():
    cfg = CONFIGS["d264k48@56"]
    ref, _ = O.ref_model_params(list(cfg.block_sizes), cfg.growth_rate, 1, cfg.compression, cfg.num_classes,
                                cfg.c0, (1, 3, 56, 56), 11)
    assert np.array_equal(init_params(cfg, 11).view(np.uint32), ref.view(np.uint32))


def test_imagenet_stem_layout():
    for name in ("d121", "d264k32", "d264k48"):
        cfg, ref56 = CONFIGS[name], CONFIGS[name + "@56"]
        pe, re_ = model_sizes(cfg)
        pe56, re56 = model_sizes(ref56)
        c0 = cfg.c0
        # 7x7 stem conv + its BN replace the reference's 3x3 stem conv
        assert pe == pe56 - c0 * 3 * 9 + c0 * 3 * 49 + 2 * c0
        assert re_ == re56 + 2 * c0
        assert re_ == O.model_running_size(cfg.block_sizes, cfg.growth_rate, cfg.compression, c0, 1)
        assert [(s.h, s.w) for s in cfg.block_shapes(64)] == [(56, 56), (28, 28), (14, 14), (7, 7)]
        assert cfg.block_shapes(64) == ref56.block_shapes(64)
    # "33M" / "73M" (BASELINE.json) hold with the ImageNet stem
    assert model_sizes(CONFIGS["d264k32"])[0] == 33_337_704
    assert model_sizes(CONFIGS["d264k48"])[0] == 72_686_632


def test_imagenet_stem_init_draw_order():
    """The 7x7 stem draws its weights where the reference draws its 3x3 stem,
    then the rest of the network continues the same Rng stream."""
    cfg = DenseNetConfig((2, 2), 4, True, 0.5, 10, 8, (3, 17, 19), stem="imagenet")
    p = init_params(cfg, 5)
    n7 = 8 * 3 * 49
    draws = O.rng_normal(5, n7 + 4)
    assert np.array_equal(p[:n7], (draws[:n7] * np.sqrt(2.0 / (3 * 49))).astype(np.float32))
    assert np.all(p[n7:n7 + 8] == 1) and np.all(p[n7 + 8:n7 + 16] == 0)
    assert p.size == model_sizes(cfg)[0]
