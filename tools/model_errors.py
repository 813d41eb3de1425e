"""Print the per-tensor normwise error of the GPU model step vs the reference golden step."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import test_model_gpu as T

for name in T.CASES:
    g = T._load(name)
    for dt in ("fp32", "bf16"):
        grads, loss, _ = T._run(g, dt)
        o, errs = 0, []
        for seg, size in T._segments(g):
            ref, got = g["grads"][o:o + size].astype(np.float64), grads[o:o + size].astype(np.float64)
            errs.append((np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30), seg))
            o += size
        errs.sort(reverse=True)
        print(f"{name} {dt}: loss {loss:.7f} ref {float(g['loss']):.7f}  worst {errs[0][1]} {errs[0][0]:.2e}, "
              f"median {np.median([e for e, _ in errs]):.2e}")
