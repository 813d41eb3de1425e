"""Build libdpb.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_1707_06990_b200.build

Objects are compiled in parallel into paper_1707_06990_b200/_build/ and
linked into paper_1707_06990_b200/_build/libdpb.so (git-ignored; travels
to the GPU box with the gpurun snapshot).  Rebuilds only what changed.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_build")
LIB = os.path.join(OUT, "libdpb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "--extended-lambda", "-Xptxas", "-warn-spills",
         f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
# DPB_PHASE_CLOCKS=1 at build time compiles the per-phase clock stamps of the
# tcgen05 engines in (tools/phase_clocks*.py, tools/tc2_clocks.py); the default
# build carries no debug reads on the kernels' critical path.
if os.environ.get("DPB_PHASE_CLOCKS"):
    FLAGS.append("-DDPB_PHASE_CLOCKS")
# DPB_EXTRA_FLAGS="-DX ..." (timing experiments only)
FLAGS += os.environ.get("DPB_EXTRA_FLAGS", "").split()


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _flags_changed() -> bool:
    """Record the compile flags; True when they differ from the last build's."""
    stamp = os.path.join(OUT, "flags.txt")
    now = " ".join(ARCH + FLAGS)
    old = open(stamp).read() if os.path.exists(stamp) else None
    if old != now:
        with open(stamp, "w") as f:
            f.write(now)
    return old != now


def _compile(src: str, verbose: bool, force: bool = False) -> str:
    obj = os.path.join(OUT, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _deps_mtime():
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose or r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    force = _flags_changed()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, force), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
