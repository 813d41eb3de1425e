"""TEST INFRASTRUCTURE — CPU timing legs of bench.py (cpu_baseline and
``--impl reference``).  Imported only by bench.py; never by the product.

Times the reference CPU implementation of the hot path — the dense-block
forward + backward of ``denseplan`` (its public ``ops::`` in GraphPlan's
order, oracle/_ref built from /root/reference by oracle/Makefile) — on the
same block shapes the GPU arm runs, with one image per process and one
process per host core (the reference is single-threaded).  When
oracle/_ref was not built, the plain-C restatement (liboracle.so) is timed
instead and reported as kind "port".

This module must not import torch: workers are spawned processes.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from oracle import oracle as O


def kind() -> str:
    return "reference" if os.path.exists(O.REF_FAST_SO) else "port"


def _worker(args):
    shapes, seed = args
    k = kind()
    cases = []
    for i, s in enumerate(shapes):
        shp = O.BlockShape(*s)
        p = O.random_block_params(shp, seed + i, np.float32)
        x = O.rng_normal(seed + 10 + i, shp.n * shp.c0 * shp.h * shp.w, np.float32).reshape(
            shp.n, shp.c0, shp.h, shp.w)
        acc = O.rng_normal(seed + 20 + i, shp.n * shp.c_out * shp.h * shp.w, np.float32).reshape(
            shp.n, shp.c_out, shp.h, shp.w)
        cases.append((shp, p, x, acc))
    t0 = time.perf_counter()
    for shp, p, x, acc in cases:
        if k == "reference":
            L = O.ref_lib(fast=True)
            feats = np.zeros((shp.n, shp.c_out, shp.h, shp.w), np.float32)
            z = np.zeros((shp.m, shp.n, shp.bk, shp.h, shp.w), np.float32)
            st = np.zeros(shp.stat_size, np.float32)
            run = shp.initial_running(np.float32)
            g = np.zeros(shp.param_size, np.float32)
            a = np.ascontiguousarray(acc)
            rc = L.ref_block_harness_f32(shp.n, shp.h, shp.w, shp.c0, shp.m, shp.k, shp.bk, O._ptr(p),
                                         O._ptr(np.ascontiguousarray(x)), O._ptr(run), 1, O._ptr(feats),
                                         O._ptr(z), O._ptr(st), O._ptr(a), O._ptr(g))
            assert rc == 0
        else:
            f, z, st, run = O.block_forward(shp, p, x)
            O.block_backward(shp, p, f, z, st, acc)
    return time.perf_counter() - t0


class CpuRunner:
    """A pool of `procs` spawned single-threaded workers; each step runs one
    image of every block shape per worker and returns (images, seconds)."""

    def __init__(self, shapes, procs: int | None = None):
        self.shapes = [tuple(s) for s in shapes]
        self.procs = procs or os.cpu_count() or 1
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.procs)
        n = self.shapes[0][0]
        self.images_per_worker = n

    def step(self, seed: int = 0):
        t0 = time.perf_counter()
        self.pool.map(_worker, [(self.shapes, seed + 1000 * i) for i in range(self.procs)])
        wall = time.perf_counter() - t0
        return self.procs * self.images_per_worker, wall

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
