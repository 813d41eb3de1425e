"""DPLN checkpoints against the reference's own writer
(checkpoint.hpp:121-198 via oracle/_ref): our reader recovers a reference
training checkpoint exactly, our writer reproduces it byte for byte, and
corruption / mismatches raise FormatError like load_checkpoint does."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1707_06990_b200 import errors
from paper_1707_06990_b200 import model as M

pytestmark = pytest.mark.skipif(not os.path.exists(O.REF_SO), reason="oracle/_ref not built")

NETS = [((2, 2, 2), 4, 0.5, 10, 8, (4, 3, 8, 8), 7), ((3, 3, 3), 12, 0.5, 10, 24, (2, 3, 16, 16), 11)]


def _cfg(blocks, k, comp, classes, c0, in_shape):
    return M.DenseNetConfig(tuple(blocks), k, True, comp, classes, c0, tuple(in_shape[1:]))


@pytest.mark.parametrize("net", NETS)
def test_reads_reference_training_checkpoint_and_rewrites_it_bytewise(tmp_path, net):
    blocks, k, comp, classes, c0, in_shape, seed = net
    ref_file = str(tmp_path / "ref.dpln")
    O.ref_save_training_checkpoint(blocks, k, comp, classes, c0, in_shape, seed, ref_file, epoch=17)
    cfg = _cfg(blocks, k, comp, classes, c0, in_shape)
    params, vel, epoch = M.load_checkpoint(cfg, ref_file, with_velocity=True)
    ref_params, _ = O.ref_model_params(blocks, k, 1, comp, classes, c0, in_shape, seed)
    assert epoch == 17
    np.testing.assert_array_equal(params.numpy(), ref_params)
    np.testing.assert_array_equal(vel.numpy(), np.float32(0.5) * ref_params)
    ours = str(tmp_path / "ours.dpln")
    M.save_checkpoint(cfg, ours, params, vel, epoch=17)
    assert open(ours, "rb").read() == open(ref_file, "rb").read()
    # parameters-only round trip
    p_only = str(tmp_path / "p.dpln")
    M.save_checkpoint(cfg, p_only, params, None, epoch=3)
    p2, v2, e2 = M.load_checkpoint(cfg, p_only)
    assert v2 is None and e2 == 3
    assert torch.equal(p2, params)


def test_corruption_and_mismatch_raise_format_error(tmp_path):
    blocks, k, comp, classes, c0, in_shape, seed = NETS[0]
    f = str(tmp_path / "ref.dpln")
    O.ref_save_training_checkpoint(blocks, k, comp, classes, c0, in_shape, seed, f, epoch=1)
    cfg = _cfg(blocks, k, comp, classes, c0, in_shape)
    raw = bytearray(open(f, "rb").read())
    bad = str(tmp_path / "bad.dpln")
    raw2 = bytearray(raw)
    raw2[100] ^= 0xFF                      # payload flip: checksum mismatch
    open(bad, "wb").write(raw2)
    with pytest.raises(errors.FormatError, match="checksum"):
        M.load_checkpoint(cfg, bad, with_velocity=True)
    open(bad, "wb").write(raw[:10])        # truncated
    with pytest.raises(errors.FormatError):
        M.load_checkpoint(cfg, bad, with_velocity=True)
    with pytest.raises(errors.FormatError, match="tensors, expected"):  # params-only vs training file
        M.load_checkpoint(cfg, f, with_velocity=False)
    other = _cfg((2, 2, 2), 4, 0.5, 10, 12, in_shape)                   # different stem width
    with pytest.raises(errors.FormatError):
        M.load_checkpoint(other, f, with_velocity=True)
    with pytest.raises(errors.FormatError, match="cannot open"):
        M.load_checkpoint(cfg, str(tmp_path / "missing.dpln"))
