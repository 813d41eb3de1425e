"""Debug: per-tile phase timing of the v2 engine (dpb_debug_tc2_clocks).
Needs a build with the stamps compiled in: rm -rf paper_1707_06990_b200/_build &&
DPB_PHASE_CLOCKS=1 python -m paper_1707_06990_b200.build (the default build has none).

    python tools/tc2_clocks.py [c] [0] [fwd|bwd] [block]      (second argument reserved)

c: the layer input width whose v2 launches stamp (default 204: BC-100 block 0,
layer 15); block: the BC-100 block geometry (0, 1, 2).  The stamps are
%globaltimer (ns, one clock for every SM), shown in us since the earliest CTA
start of the recorded launch.  'fwd' records the layer's 1x1 forward; by
default the backward runs last and its 1x1 dgrad's stamps are read.
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1707_06990_b200 as P  # noqa: E402
from paper_1707_06990_b200._lib import lib  # noqa: E402
from bench import block_shapes  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 204
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
fwd_only = len(sys.argv) > 3 and sys.argv[3] == "fwd"
blk = int(sys.argv[4]) if len(sys.argv) > 4 else 0
L = lib()
f = L.dpb_debug_tc2_clocks
f.argtypes = [C.c_int, C.c_void_p]
import os  # noqa: E402
shp = P.BlockShape(*block_shapes(os.environ.get("CFG", "bc100"), 64)[blk])
plan = P.BlockPlan(shp, dtype="bf16", layout="nhwc")
p = torch.randn(shp.param_elems, device="cuda") * 0.1 + 0.5
x = torch.randn(shp.pixels, shp.c0, device="cuda")
run = shp.initial_running()
acc = torch.randn(shp.pixels, shp.c_out, device="cuda")
grads = torch.empty(shp.param_elems, device="cuda")
for _ in range(2):
    plan.forward(x, p, run, True)
    plan.backward(p, acc.clone(), grads)
torch.cuda.synchronize()
f(c | (flags << 16), None)
plan.forward(x, p, run, True)
if not fwd_only:
    plan.backward(p, acc.clone(), grads)
torch.cuda.synchronize()
f(0, None)
buf = np.zeros((148, 28), dtype=np.int64)
f(0, C.c_void_p(buf.ctypes.data))
valid = buf[:, 0] > 0
t0 = buf[valid, 0].min()
rel = (buf - t0) / 1e3
np.set_printoptions(linewidth=200, precision=2, suppress=True)
print(f"block {blk} {shp}, c={c}, {'fwd' if fwd_only else 'bwd'}: {valid.sum()} CTAs stamped; "
      f"us since the first CTA start")
names = ["start", "prologue"] + [f"tma{t}" for t in range(4)] + [f"xf{t}" for t in range(4)] + \
        [f"mma{t}" for t in range(4)] + [f"epi_s{t}" for t in range(4)] + [f"epi_e{t}" for t in range(4)] + ["exit"]
for i, n in enumerate(names[:23]):
    m = valid & (buf[:, i] > 0)
    col = rel[m, i]
    if len(col):
        print(f"{n:9s} mean {col.mean():7.2f}  min {col.min():7.2f}  max {col.max():7.2f}  cta0 {rel[0, i]:7.2f}")
print("epi_full wait us per CTA: warp2 mean %.2f, warp6 mean %.2f" % (buf[valid, 23].mean() / 1e3,
                                                                      buf[valid, 24].mean() / 1e3))
print("xf wait us per CTA: raw_full %.2f, op_empty %.2f; tma wait raw_empty %.2f" % (
    buf[valid, 25].mean() / 1e3, buf[valid, 26].mean() / 1e3, buf[valid, 27].mean() / 1e3))
