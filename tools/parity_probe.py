"""Diagnostic: per-tensor error of a whole training step against the float64
reference sketch of a TRAIN_CASES fixture (tests/golden/train_*.npz).
Usage: python tools/parity_probe.py train_d264k32_56 fp32"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_train_gpu as T  # noqa: E402
from oracle import oracle as O  # noqa: E402

name, dtype = sys.argv[1], sys.argv[2]
g = T._load(name)
grads, loss, running = T._run(g, dtype)
gsegs, rsegs = T._segs(g)
print("loss", loss, "ref64", float(g["loss64"]), "ref32", float(g["loss"]))
for what, got, segs in (("grads", grads, gsegs), ("running", running, rsegs)):
    ref = {k[len(what) + 3:]: v for k, v in g.items() if k.startswith(what + "64_")}
    est, rel = O.sketch_errors(got, ref, segs)
    nw = g[what + "_noise"]
    order = np.argsort(-est / np.maximum(nw, 1e-12))
    tot = np.sqrt(np.sum((est * ref["norm"]) ** 2)) / np.sqrt(np.sum(ref["norm"] ** 2))
    print(f"== {what}: whole-vector {tot:.3e}; median est {np.median(est):.3e} median noise {np.median(nw):.3e}")
    for i in order[:25]:
        print(f"  {segs[i][0]:28s} n={segs[i][1]:8d} est={est[i]:.3e} noise={nw[i]:.3e} norm={ref['norm'][i]:.3e}")
    # error by position
    byb = {}
    for i, (sname, _) in enumerate(segs):
        key = sname.split(".")[0]
        byb.setdefault(key, []).append(est[i])
    print("  per group median:", {k: f"{np.median(v):.2e}" for k, v in byb.items()})
