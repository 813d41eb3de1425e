"""Debug: per-tile phase timing of the v2 engine (dpb_debug_tc2_clocks).

    python tools/tc2_clocks.py [c]      # c = layer width to record (default 204: BC-100 block 1, layer 15)

Runs the BC-100 block-1 geometry (64x32x32, c0=24, m=16, k=12, bk=48) forward
and backward; the v2 launches of the layer with input width c stamp clock64()
per CTA (see dpb_tc2.cuh).  Both the 1x1 forward and the 1x1 dgrad of that
layer match; the backward runs last, so the dgrad's stamps are what is read.
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1707_06990_b200 as P  # noqa: E402
from paper_1707_06990_b200._lib import lib  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 204
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # A/B: 1 skip g1 stores, 2 skip column sums
fwd_only = len(sys.argv) > 3 and sys.argv[3] == "fwd"  # stamps of the layer's last forward launch (3x3)
L = lib()
f = L.dpb_debug_tc2_clocks
f.argtypes = [C.c_int, C.c_void_p]
shp = P.BlockShape(64, 32, 32, 24, 16, 12, 48)
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
rel = (buf - buf[:, :1]) / 1.965e3  # per-CTA clocks (not synchronised across SMs) -> us
np.set_printoptions(linewidth=200, precision=1, suppress=True)
print("per-CTA timeline (us since the CTA's own start), mean over CTAs / CTA 0:")
names = ["start", "prologue"] + [f"tma{t}" for t in range(4)] + [f"xf{t}" for t in range(4)] + \
        [f"mma{t}" for t in range(4)] + [f"epi_s{t}" for t in range(4)] + [f"epi_e{t}" for t in range(4)] + ["exit"]
valid = buf[:, 0] > 0
for i, n in enumerate(names[:23]):
    col = rel[valid, i]
    col = col[buf[valid, i] > 0]
    if len(col):
        print(f"{n:9s} mean {col.mean():7.2f}  min {col.min():7.2f}  max {col.max():7.2f}  cta0 {rel[0, i]:7.2f}")
print("epi_full wait us per CTA: warp2 mean %.2f, warp6 mean %.2f" % (buf[valid, 23].mean() / 1.965e3, buf[valid, 24].mean() / 1.965e3))
