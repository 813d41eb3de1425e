"""HostBlockChain (host-buffer step, copy stream + per-block events) against the
same blocks driven directly through BlockPlan: bitwise equal gradients and
block-input gradients over consecutive steps with changing inputs."""
import numpy as np
import pytest
import torch

import paper_1707_06990_b200 as P
from paper_1707_06990_b200.host import HostBlockChain

pytestmark = pytest.mark.gpu

SHAPES = [(4, 16, 16, 24, 4, 12, 48), (4, 8, 8, 36, 3, 12, 48)]


def _params(shp, g):
    p = torch.randn(shp.param_elems, generator=g) * 0.1
    for l, o in enumerate(shp.param_offsets()):
        c = shp.c_in(l)
        p[o:o + c] += 1.0
        gb = o + 2 * c + shp.bk * c
        p[gb:gb + shp.bk] += 1.0
    return p.cuda()


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_chain_matches_direct_calls(dtype):
    g = torch.Generator().manual_seed(5)
    shapes = [P.BlockShape(*s) for s in SHAPES]
    params = [_params(s, g) for s in shapes]
    run_chain = [s.initial_running("cuda") for s in shapes]
    run_direct = [s.initial_running("cuda") for s in shapes]
    chain = HostBlockChain(shapes, params, run_chain, dtype=dtype, layout="nchw")
    direct = [P.BlockPlan(s, dtype=dtype, layout="nchw") for s in shapes]
    for step in range(3):
        xs = [torch.randn(s.n, s.c0, s.h, s.w, generator=g).pin_memory() for s in shapes]
        gs = [torch.randn(s.n, s.c_out, s.h, s.w, generator=g).pin_memory() for s in shapes]
        host = chain.step(xs, gs)
        chain.stream.synchronize()
        got = host.clone()
        want = []
        accs = []
        for b, s in enumerate(shapes):
            direct[b].forward(xs[b].cuda(), params[b], run_direct[b], True)
        for b in reversed(range(len(shapes))):
            acc = gs[b].cuda()
            grads = torch.empty(shapes[b].param_elems, device="cuda")
            direct[b].backward(params[b], acc, grads)
            want.insert(0, grads)
            accs.insert(0, acc)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.numpy(), torch.cat(want).cpu().numpy(), err_msg=f"step {step}")
        for b in range(len(shapes)):
            np.testing.assert_array_equal(chain.acc[b].cpu().numpy(), accs[b].cpu().numpy())
            np.testing.assert_array_equal(run_chain[b].cpu().numpy(), run_direct[b].cpu().numpy())
    chain.close()
    for d in direct:
        d.close()
