"""Per-parameter-group parity breakdown of the block path vs the f64 oracle."""
import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_block_gpu import oracle_case, run_device
from oracle import oracle as O

def breakdown(s, dtype, seed=7):
    ref = oracle_case(s, seed)
    got = run_device(s, ref["params"], ref["x_in"], ref["running_in"], ref["acc_in"], dtype)
    shp = O.BlockShape(*s)
    g, r = got["grads"], ref["f64"]["grads"]
    out = []
    for l, o in enumerate(shp.param_offsets()):
        c, bk, k = shp.c_in(l), shp.bk, shp.k
        parts = {"ga": (o, c), "ba": (o + c, c), "w1": (o + 2 * c, bk * c), "gb": (o + 2 * c + bk * c, bk),
                 "bb": (o + 2 * c + bk * c + bk, bk), "w2": (o + 2 * c + bk * c + 2 * bk, 9 * k * bk)}
        errs = {kk: float(np.linalg.norm(g[a:a + n] - r[a:a + n]) / (np.linalg.norm(r[a:a + n]) + 1e-30))
                for kk, (a, n) in parts.items()}
        out.append(f"l{l}: " + " ".join(f"{kk}={v:.1e}" for kk, v in errs.items()))
    acc_e = np.linalg.norm(got["acc_out"] - ref["f64"]["acc_out"]) / np.linalg.norm(ref["f64"]["acc_out"])
    print(s, dtype, "acc", f"{acc_e:.2e}")
    print("\n".join(out[-3:] + out[:2]))

if __name__ == "__main__":
  for s in [(16, 32, 32, 24, 2, 12, 48), (4, 32, 32, 24, 12, 12, 48), (16, 16, 16, 24, 12, 12, 48)]:
      breakdown(s, "fp32")
