"""Momentum SGD and learning-rate schedules.

CPU: the restatement pinned to the reference (oracle/_ref) bitwise, and the
library's dpb_lr_at against the reference's lr_at.  GPU: dpb_sgd_step against
the reference's sgd_step, bitwise (the kernel rounds every product and sum
like the reference's float loop)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1707_06990_b200 import errors, ops

HAVE_REF = os.path.exists(O.REF_SO)
CASES = [(0.1, 0.9, 1e-4, False), (0.05, 0.9, 5e-4, True), (1.0, 0.0, 0.0, False)]


def _data(n, seed):
    r = np.random.default_rng(seed)
    return (r.standard_normal(n).astype(np.float32), r.standard_normal(n).astype(np.float32),
            r.standard_normal(n).astype(np.float32))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("lr,mu,wd,nest", CASES)
def test_restatement_matches_reference_sgd_bitwise(lr, mu, wd, nest):
    p, g, v = _data(1000, 3)
    p2, v2 = p.copy(), v.copy()
    for _ in range(3):
        O.sgd_step(p, g, v, lr, mu, wd, nest)
        O.ref_sgd_step(p2, g, v2, lr, mu, wd, nest)
    np.testing.assert_array_equal(p, p2)
    np.testing.assert_array_equal(v, v2)


def test_lr_schedules():
    for epoch in range(0, 90, 7):
        want = O.lr_at("step", 0.1, 90, epoch, (30, 60), 0.1)
        assert ops.lr_at("step", 0.1, 90, epoch, (30, 60), 0.1) == pytest.approx(want, rel=1e-15)
        want = O.lr_at("cosine", 0.1, 90, epoch, floor=1e-3)
        assert ops.lr_at("cosine", 0.1, 90, epoch, floor=1e-3) == pytest.approx(want, rel=1e-15)
        if HAVE_REF:
            assert ops.lr_at("step", 0.1, 90, epoch, (30, 60), 0.1) == O.ref_lr_at("step", 0.1, 90, epoch, (30, 60), 0.1)
            assert ops.lr_at("cosine", 0.1, 90, epoch, floor=1e-3) == O.ref_lr_at("cosine", 0.1, 90, epoch, floor=1e-3)
    with pytest.raises(errors.RangeError):
        ops.lr_at("step", 0.1, 90, 90)


@pytest.mark.gpu
@pytest.mark.parametrize("lr,mu,wd,nest", CASES)
def test_sgd_step_matches_reference_bitwise(lr, mu, wd, nest):
    import torch
    n = 100_003  # not a multiple of the block size
    p, g, v = _data(n, 7)
    tp, tg, tv = (torch.from_numpy(a.copy()).cuda() for a in (p, g, v))
    for _ in range(3):
        ops.sgd_step(tp, tg, tv, lr, mu, wd, nest)
        O.sgd_step(p, g, v, lr, mu, wd, nest)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(tp.cpu().numpy(), p)
    np.testing.assert_array_equal(tv.cpu().numpy(), v)
