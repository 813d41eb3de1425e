"""TEST INFRASTRUCTURE — CPU timing legs of bench.py (cpu_baseline and
``--impl reference``).  Imported only by bench.py; never by the product.

Times the reference CPU implementation, built from /root/reference by
oracle/Makefile into oracle/_ref, with one process per host core (the
reference is single-threaded):

- CpuModelRunner: the whole training step, GraphPlan<float>::step_trace (the
  reference's public API), on the same network the GPU arm runs, with a small
  batch per process.
- CpuRunner: the dense-block forward + backward alone (the reference's public
  ops:: in GraphPlan's order), one image of each block shape per process.
  When oracle/_ref was not built, the plain-C restatement (liboracle.so) is
  timed instead and reported as kind "port".

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


def _model_worker(args):
    net, batch, seed = args
    blocks, k, comp, classes, c0, in_shape = net
    loss, secs = O.ref_model_step(blocks, k, 1, comp, classes, c0, (batch,) + tuple(in_shape), seed,
                                  steps=1, fast=True)
    return secs


class CpuModelRunner:
    """`procs` spawned single-threaded workers, each timing one reference
    training step (GraphPlan::step_trace) of the network at `batch` images;
    a step returns (images, seconds of the slowest worker's step)."""

    def __init__(self, net, batch: int = 1, procs: int | None = None):
        if kind() != "reference":
            raise FileNotFoundError("oracle/_ref (the reference build) is required for the model runner")
        self.net = net
        self.batch = batch
        self.procs = procs or os.cpu_count() or 1
        self.pool = mp.get_context("spawn").Pool(self.procs)

    def step(self, seed: int = 0):
        secs = self.pool.map(_model_worker, [(self.net, self.batch, seed + i) for i in range(self.procs)])
        return self.procs * self.batch, max(secs)

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
