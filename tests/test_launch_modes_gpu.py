"""The launch path does not change results (GPU).

Every block-path kernel uses programmatic dependent launch, and several read
data written two or more launches back before their grid-dependency wait:
resident weight images, the first TMA ring stages, BN tables from forward
statistics, and the first rows of the BN_a apply.  The backward forks its
weight gradients onto a side stream.  The same training step (three steps,
graph-replayed) must give bitwise-identical gradients, loss and running
statistics in three modes: default, without PDL (every launch fully
serialised), and without PDL or the side stream.  Each mode runs in its own
process, because the switches are read once per process.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp_path, name, env_extra):
    out = tmp_path / f"{name}.npz"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_launch_probe.py"), str(out)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def test_launch_modes_are_bit_identical(tmp_path):
    base = _run(tmp_path, "default", {})
    for name, env in (("no_pdl", {"DPB_NO_PDL": "1"}), ("serial", {"DPB_NO_PDL": "1", "DPB_NO_FORK": "1"})):
        got = _run(tmp_path, name, env)
        for key in ("grads", "loss", "running"):
            assert np.isfinite(got[key]).all(), (name, key)
            assert np.array_equal(base[key], got[key]), f"{key} differs between default and {name} launches"
