"""The OpTrace contract (alloctrace.hpp:132-201; t/graph_test.cpp:249-298) on
the reference itself: which nodes a SharedAll step recomputes, and the FLOP
conventions (ops.hpp:565-595) that tests/test_trace_gpu.py holds the device
block's trace to (oracle.block_trace_flops)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

HAVE_REF = os.path.exists(O.REF_SO)
KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kats.json")))


def _ref(strategy=2):
    if strategy == 2:
        t = KATS["block_trace_m3k4c8_n2h5w6"]
        return np.array(t["counts"]), np.array(t["flops"])
    if not HAVE_REF:
        pytest.skip("oracle/_ref not built")
    return O.ref_single_block_trace(3, 4, 8, 2, 5, 6, strategy=strategy)


def test_reference_recomputes_concat_bn_relu_once_per_layer():
    counts, _ = _ref()
    m = 3
    for l in range(m):
        base = 1 + 7 * l  # node 0 is the stem conv
        for j, kind in enumerate(["concat", "bn_a", "relu_a", "conv_a", "bn_b", "relu_b", "conv_b"]):
            f, b, r = counts[base + j]
            assert f == 1 and b == 1, (l, kind)
            assert r == (0 if kind.startswith("conv") else 1), (l, kind)


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_reference_naive_never_recomputes():
    counts, flops = _ref(strategy=0)
    assert counts[:, 2].sum() == 0 and flops[2].sum() == 0.0


def test_flop_conventions_match_reference_totals():
    """oracle.block_trace_flops + the stem / head terms == the reference's totals."""
    _, flops = _ref()
    s = O.BlockShape(2, 5, 6, 8, 3, 4, 16)
    fwd, bwd, rem = block_trace_flops = O.block_trace_flops(s)
    M, C = 2 * 5 * 6, s.c_out
    stem = 2.0 * M * 8 * 3 * 9                      # 3x3 stem conv
    assert flops[0][0] == fwd[0]                    # concats (layer + block output)
    assert flops[0][1] == fwd[1] + 8.0 * M * C      # + head BN
    assert flops[0][2] == fwd[2] + M * C            # + head ReLU
    assert flops[0][3] == fwd[3] + stem
    assert flops[1][1] == bwd[1] + 12.0 * M * C
    assert flops[1][3] == bwd[3] + 2.0 * stem
    assert flops[2][0] == rem[0] + M * C            # + the head's re-concat of the block output
    assert flops[2][1] == rem[1] + 8.0 * M * C
    assert flops[2][2] == rem[2] + M * C
    assert flops[2][3] == 0.0
