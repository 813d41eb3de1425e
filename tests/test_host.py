"""Host-side logic of the product library (CPU only, no device calls):
the C ABI loads and exports every declared symbol, the model arithmetic and
arena plan are bit-exact against the reference's known answers, and errors
map to the reference's exception classes."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
import paper_1707_06990_b200 as P
from paper_1707_06990_b200 import errors, model
from paper_1707_06990_b200._lib import SIGNATURES, BlockDesc, ArenaSizes, lib

KATS = json.load(open(os.path.join(GOLDEN, "kats.json")))


def declared_symbols():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            names |= set(re.findall(r"DPB_API\s+[\w\s\*]*?\b(dpb_\w+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 20
    L = lib()
    for n in sorted(names):
        assert hasattr(L, n), n
    assert names == set(SIGNATURES), names ^ set(SIGNATURES)


def test_version_string():
    assert b"sm_100a" in lib().dpb_version()


@pytest.mark.parametrize("name,cfg", [
    ("bc100_k12", model.DenseNetConfig((16, 16, 16), 12, True, 0.5, 10, 24)),
    ("d121_k32", model.DenseNetConfig((6, 12, 24, 16), 32, True, 0.5, 1000, 64)),
    ("d264_k32", model.DenseNetConfig((6, 12, 64, 48), 32, True, 0.5, 1000, 64)),
    ("d264_k48", model.DenseNetConfig((6, 12, 64, 48), 48, True, 0.5, 1000, 96)),
    ("bc160_k12", model.DenseNetConfig((26, 26, 26), 12, True, 0.5, 10, 24)),
    ("paper264_k48_preset", model.DenseNetConfig((6, 32, 64, 48), 48, True, 0.5, 1000, 96)),
    ("paper264_k32_preset", model.DenseNetConfig((6, 32, 64, 48), 32, True, 0.5, 1000, 64)),
])
def test_count_parameters_matches_reference(name, cfg):
    assert model.count_parameters(cfg) == KATS["count_parameters"][name]


def test_frozen_parameter_counts():
    # t/densenet_test.cpp:214-231 and BASELINE.json's 33M / 73M
    assert KATS["count_parameters"]["paper264_k48_preset"] == 90500680
    assert KATS["count_parameters"]["bc160_k12"] == 1739002
    assert KATS["count_parameters"]["d264_k32"] == 33329896
    assert KATS["count_parameters"]["d264_k48"] == 72674920


PEAK_CFGS = {
    "tiny_block_k2": (model.DenseNetConfig((3,), 2, False, 1.0, 2, 2), 1, 1, 4, 4),
    "cfg1": (model.DenseNetConfig((12,), 12, True, 1.0, 10, 24), 16, 3, 32, 32),
    "bc100_b64": (model.DenseNetConfig((16, 16, 16), 12, True, 0.5, 10, 24), 64, 3, 32, 32),
    "d121_b64_56": (model.DenseNetConfig((6, 12, 24, 16), 32, True, 0.5, 1000, 64), 64, 3, 56, 56),
    "d264k32_b64_56": (model.DenseNetConfig((6, 12, 64, 48), 32, True, 0.5, 1000, 64), 64, 3, 56, 56),
    "d264k48_b64_56": (model.DenseNetConfig((6, 12, 64, 48), 48, True, 0.5, 1000, 96), 64, 3, 56, 56),
}


@pytest.mark.parametrize("name", sorted(PEAK_CFGS))
@pytest.mark.parametrize("strategy", ["naive", "shared_grad", "shared_all"])
def test_predict_peak_elements_matches_reference(name, strategy):
    cfg, n, c, h, w = PEAK_CFGS[name]
    got = model.predict_peak_elements(cfg, strategy.replace("_", "-"), n, c, h, w)
    assert [got[a] for a in model.ARENAS] == KATS["predict_peak_elements"][name][strategy]


def test_peak_model_hand_enumerated_kat():
    # t/alloctrace_test.cpp:85-124
    cfg = model.DenseNetConfig((3,), 2, False, 1.0, 2, 2)
    naive = model.predict_peak_elements(cfg, "naive", 1, 1, 4, 4)
    sa = model.predict_peak_elements(cfg, "shared-all", 1, 1, 4, 4)
    assert naive["feature_owned"] == 1426 and naive["scratch"] == 2
    assert (sa["feature_owned"], sa["shared1"], sa["shared2"], sa["shared_grad"]) == (138, 128, 128, 512)
    assert sa["params"] == 2 * 292


def test_rng_matches_reference_draws():
    np.testing.assert_array_equal(model.rng_normal(106, 8),
                                  np.array(KATS["rng_normal_seed106_first8"], dtype=np.float32))


def test_arena_plan_offsets_and_sizes_exact():
    s = P.BlockShape(16, 32, 32, 24, 12, 12, 48)   # cfg1
    M, C, cmax = 16 * 32 * 32, 24 + 12 * 12, 24 + 11 * 12
    for dtype, S in (("fp32", 4), ("bf16", 4)):
        a = P.plan_arena(s, dtype, "nchw")
        assert a["feat_offset"] == 0 and a["feat_bytes"] == M * C * S
        assert a["z_bytes"] == 12 * M * 48 * S
        assert a["acc_bytes"] == M * C * 4
        # g0 is double-buffered across layers (two-stream backward)
        assert a["g0_bytes"] == 2 * M * 48 * 4 and a["g1_bytes"] == 2 * M * cmax * 4
        assert a["shared1_bytes"] == 0 and a["shared2_bytes"] == 0
        assert a["param_elems"] == s.param_elems and a["stat_elems"] == s.stat_elems
        # regions are 256-byte aligned, ordered and disjoint
        regs = [(a[f"{r}_offset"], a[f"{r}_bytes"]) for r in
                ("feat", "z", "stats", "acc", "g0", "g1", "scratch")]
        for (o1, b1), (o2, _) in zip(regs, regs[1:]):
            assert o1 % 256 == 0 and o2 >= o1 + b1
        assert a["total_bytes"] >= regs[-1][0] + regs[-1][1]
    # NHWC boundary: the caller's gradient buffer is the accumulator
    assert P.plan_arena(s, "bf16", "nhwc")["acc_bytes"] == 0


def test_block_memory_is_linear_vs_naive_quadratic():
    effs, naives = [], []
    for m in (8, 16, 32, 64):
        e, n = P.block_memory(P.BlockShape(8, 16, 16, 24, m, 12, 48), "fp32")
        effs.append(e)
        naives.append(n)
    # doubling depth: efficient grows ~2x (O(m)), naive ~>3x (O(m^2))
    assert effs[-1] / effs[-2] < 2.3
    assert naives[-1] / naives[-2] > 3.0


@pytest.mark.parametrize("field,value,exc", [
    ("n", 0, errors.ShapeError), ("c0", 0, errors.ShapeError), ("dtype", 7, errors.ConfigError),
    ("layout", 3, errors.ConfigError), ("n", 1 << 56, errors.SizeOverflowError)])
def test_plan_rejects_bad_descriptors(field, value, exc):
    d = BlockDesc(2, 4, 4, 8, 2, 4, 16, 0, 0)
    setattr(d, field, value)
    s = ArenaSizes()
    from paper_1707_06990_b200._lib import check
    with pytest.raises(exc):
        check(lib().dpb_block_plan(C.byref(d), C.byref(s)))


def test_config_errors():
    with pytest.raises(errors.ConfigError):
        model.count_parameters(model.DenseNetConfig((0,), 12))
    with pytest.raises(errors.ConfigError):
        model.count_parameters(model.DenseNetConfig((4,), 12, compression=1.5))


def test_block_shapes_match_geometry():
    shapes = model.CONFIGS["d264k48"].block_shapes(64)
    assert [(s.h, s.c0, s.m) for s in shapes] == [(56, 96, 6), (28, 192, 12), (14, 384, 64), (7, 1728, 48)]
    assert shapes[2].c_out == 384 + 64 * 48 == 3456
    bc = model.CONFIGS["bc100"].block_shapes(64)
    assert [(s.h, s.c0, s.c_out) for s in bc] == [(32, 24, 216), (16, 108, 300), (8, 150, 342)]


def test_model_sizes_match_reference_parameter_count():
    # dpb_model_sizes (registration-order layout) == densenet.hpp count_parameters
    from paper_1707_06990_b200.model import CONFIGS, DenseNetConfig, ModelPlan  # noqa: F401
    import ctypes as C
    from paper_1707_06990_b200._lib import ModelDesc, lib
    cases = [DenseNetConfig((2, 2, 2), 4, True, 0.5, 10, 8, (3, 8, 8)),
             DenseNetConfig((3, 3, 3), 12, True, 0.5, 10, 24, (3, 16, 16)),
             CONFIGS["bc100"]]
    for cfg in cases:
        d = ModelDesc()
        d.nblocks = len(cfg.block_sizes)
        for i, m in enumerate(cfg.block_sizes):
            d.blocks[i] = m
        d.k, d.compression, d.classes, d.c0 = cfg.growth_rate, cfg.compression, cfg.num_classes, cfg.c0
        d.in_c, d.in_h, d.in_w = cfg.in_shape
        d.batch, d.dtype = 4, 1
        pe, re_ = C.c_int64(), C.c_int64()
        assert lib().dpb_model_sizes(C.byref(d), C.byref(pe), C.byref(re_)) == 0
        assert pe.value == P.count_parameters(cfg)
        # running: per block its stats, per transition / head 2C
        shapes = cfg.block_shapes(4)
        assert re_.value == sum(s.stat_elems + 2 * s.c_out for s in shapes)


def test_model_sizes_rejects_bad_geometry():
    import ctypes as C
    from paper_1707_06990_b200._lib import ModelDesc, lib
    d = ModelDesc()
    d.nblocks, d.k, d.compression, d.classes, d.c0 = 2, 4, 0.0, 10, 8
    d.blocks[0] = d.blocks[1] = 2
    d.in_c, d.in_h, d.in_w, d.batch = 3, 8, 8, 2
    assert lib().dpb_model_sizes(C.byref(d), None, None) == 6      # ConfigError (compression)
    d.compression, d.nblocks = 0.5, 0
    assert lib().dpb_model_sizes(C.byref(d), None, None) == 6


def test_naive_block_rejects_unknown_strategy():
    from paper_1707_06990_b200.naive import NaiveBlock
    with pytest.raises(ValueError):
        NaiveBlock(P.BlockShape(1, 4, 4, 8, 2, 4, 16), "shared-all")
