"""The device block's OpTrace (dpb_block_trace) against the reference's
(tests/golden/kats.json block_trace_*, from GraphPlan::step_trace; the FLOP
conventions pinned in tests/test_trace.py).

Forward and backward counts are the reference's, node for node.  Recompute
differs by design: the concat is a zero-copy channel prefix (never copied,
never recomputed, 0 FLOPs), and act_a = relu(bn_a(cat)) and act_b =
relu(bn_b(z)) are recomputed inside the kernels' prologues twice per layer —
once for the data-gradient ReLU mask, once as the weight-gradient operand —
instead of once into Shared1/Shared2: 2x the reference's BN/ReLU recompute
FLOPs, no recompute storage.  Convolutions are never recomputed (both)."""
import json
import os

import numpy as np
import pytest
import torch

import paper_1707_06990_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu
KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kats.json")))


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_block_trace_matches_reference_contract(dtype):
    ref = np.array(KATS["block_trace_m3k4c8_n2h5w6"]["counts"])
    shp = P.BlockShape(2, 5, 6, 8, 3, 4, 16)
    plan = P.BlockPlan(shp, dtype=dtype, layout="nchw")
    g = torch.Generator().manual_seed(1)
    p = (torch.randn(shp.param_elems, generator=g) * 0.2 + 0.5).cuda()
    x = torch.randn(shp.n, shp.c0, shp.h, shp.w, generator=g).cuda()
    acc = torch.randn(shp.n, shp.c_out, shp.h, shp.w, generator=g).cuda()
    grads = torch.empty_like(p)
    plan.forward(x, p, shp.initial_running("cuda"), True)
    plan.backward(p, acc, grads)
    plan.sync()
    t = plan.trace()
    ours = t["nodes"]
    assert ours.shape[0] == 7 * shp.m + 1
    ref_block = ref[1:1 + 7 * shp.m + 1]   # node 0: the reference's stem conv
    np.testing.assert_array_equal(ours[:, 0], ref_block[:, 0])          # forward
    np.testing.assert_array_equal(ours[:-1, 1], ref_block[:-1, 1])      # backward (layers)
    for l in range(shp.m):
        for j, kind in enumerate(["concat", "bn_a", "relu_a", "conv_a", "bn_b", "relu_b", "conv_b"]):
            r = ref_block[7 * l + j, 2]
            expect = 0 if kind == "concat" else 2 * r
            assert ours[7 * l + j, 2] == expect, (l, kind)
    fwd, bwd, rem = O.block_trace_flops(shp)
    kinds = ["concat", "batchnorm", "relu", "conv"]
    for i, k in enumerate(kinds):
        assert t["forward_flops"][k] == (0.0 if k == "concat" else fwd[i]), k
        assert t["backward_flops"][k] == bwd[i], k
        assert t["recompute_flops"][k] == (0.0 if k == "concat" else 2 * rem[i]), k
    plan.close()
