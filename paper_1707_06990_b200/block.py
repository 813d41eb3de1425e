"""Host-side mirror of the reference's dense-block path over the C ABI.

``BlockPlan`` plays the role of the dense-block share of ``GraphPlan<T>``
(/root/reference/proj/include/denseplan/graph.hpp): ``build`` sizes the
shared storage once (graph.hpp:405-613), ``forward`` runs the layer loop of
``forward_layer`` (graph.hpp:618-670, 747-760) and ``backward`` runs
``backward_block`` / ``backward_layer`` with rematerialisation
(graph.hpp:1054-1063, 856-945, 831-854).  Tensors are torch CUDA tensors
used purely as device memory; every computation happens in libdpb.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import errors
from ._lib import ArenaSizes, BlockDesc, KernelStat, check, lib

FP32, BF16 = 0, 1
NCHW, NHWC = 0, 1
_DT = {"fp32": FP32, "float32": FP32, "bf16": BF16, "bfloat16": BF16}
_LAYOUT = {"nchw": NCHW, "nhwc": NHWC}


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise errors.ConfigError("device tensor expected")
    if not t.is_contiguous():
        raise errors.ShapeError("contiguous tensor expected")
    return C.c_void_p(t.data_ptr())


@dataclass(frozen=True)
class BlockShape:
    """Geometry of one dense block (densenet.hpp:124-180, bk = 4k at :68)."""
    n: int
    h: int
    w: int
    c0: int
    m: int
    k: int
    bk: int

    @property
    def c_out(self) -> int:
        return self.c0 + self.m * self.k

    def c_in(self, l: int) -> int:
        return self.c0 + l * self.k

    @property
    def pixels(self) -> int:
        return self.n * self.h * self.w

    def param_offsets(self) -> list[int]:
        offs, o = [], 0
        for l in range(self.m):
            offs.append(o)
            c = self.c_in(l)
            o += 2 * c + self.bk * c + 2 * self.bk + 9 * self.k * self.bk
        return offs

    @property
    def param_elems(self) -> int:
        c = self.c_in(self.m - 1)
        return self.param_offsets()[-1] + 2 * c + self.bk * c + 2 * self.bk + 9 * self.k * self.bk

    def stat_offsets(self) -> list[int]:
        offs, o = [], 0
        for l in range(self.m):
            offs.append(o)
            o += 2 * self.c_in(l) + 2 * self.bk
        return offs

    @property
    def stat_elems(self) -> int:
        return sum(2 * self.c_in(l) + 2 * self.bk for l in range(self.m))

    def initial_running(self, device="cuda") -> torch.Tensor:
        """Running mean 0 / var 1 (graph.hpp:358-360)."""
        r = torch.zeros(self.stat_elems, dtype=torch.float32)
        for l, o in enumerate(self.stat_offsets()):
            c = self.c_in(l)
            r[o + c:o + 2 * c] = 1
            r[o + 2 * c + self.bk:o + 2 * c + 2 * self.bk] = 1
        return r.to(device)

    def desc(self, dtype: str, layout: str) -> BlockDesc:
        return BlockDesc(self.n, self.h, self.w, self.c0, self.m, self.k, self.bk,
                         _DT[dtype], _LAYOUT[layout])


def plan_arena(shape: BlockShape, dtype: str = "bf16", layout: str = "nchw") -> dict:
    """Host-only arena plan (PoolRegion/GradPool sizing analogue)."""
    d = shape.desc(dtype, layout)
    s = ArenaSizes()
    check(lib().dpb_block_plan(C.byref(d), C.byref(s)))
    return s.as_dict()


def block_memory(shape: BlockShape, dtype: str = "bf16") -> tuple[int, int]:
    """(efficient arena bytes, naive store-everything bytes) of one block."""
    d = shape.desc(dtype, "nhwc")
    e, n = C.c_int64(), C.c_int64()
    check(lib().dpb_block_memory(C.byref(d), C.byref(e), C.byref(n)))
    return e.value, n.value


class BlockPlan:
    """One dense block bound to a GPU and a stream, owning its HBM arena."""

    def __init__(self, shape: BlockShape, dtype: str = "fp32", layout: str = "nchw",
                 device: int | None = None, stream: torch.cuda.Stream | None = None):
        self.shape = shape
        self.dtype = dtype
        self.layout = layout
        self.device = torch.cuda.current_device() if device is None else device
        self._desc = shape.desc(dtype, layout)
        self._stream = stream
        h = C.c_void_p()
        s = None if stream is None else C.c_void_p(stream.cuda_stream)
        check(lib().dpb_block_create(C.byref(self._desc), self.device, s, C.byref(h)))
        self._h = h

    @staticmethod
    def build(shape: BlockShape, **kw) -> "BlockPlan":
        return BlockPlan(shape, **kw)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().dpb_block_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: torch.cuda.Stream | None) -> None:
        self._stream = stream
        check(lib().dpb_block_set_stream(self._h, None if stream is None else C.c_void_p(stream.cuda_stream)))

    @property
    def arena(self) -> dict:
        s = ArenaSizes()
        check(lib().dpb_block_arena(self._h, C.byref(s), None))
        return s.as_dict()

    @property
    def launch_count(self) -> int:
        return int(lib().dpb_block_launch_count(self._h))

    # -- execution ------------------------------------------------------------

    def forward(self, x_in: torch.Tensor, params: torch.Tensor, running: torch.Tensor | None,
                update_running: bool = True) -> None:
        """Train-mode forward; features / z / stats stay in the arena."""
        check(lib().dpb_block_forward(self._h, _ptr(x_in), _ptr(params), _ptr(running),
                                      int(update_running)))

    def forward_eval(self, x_in: torch.Tensor, params: torch.Tensor, running: torch.Tensor) -> None:
        check(lib().dpb_block_forward_eval(self._h, _ptr(x_in), _ptr(params), _ptr(running)))

    def backward(self, params: torch.Tensor, grad_acc: torch.Tensor, grads: torch.Tensor) -> None:
        """grad_acc in/out (block-gradient accumulator); grads written."""
        check(lib().dpb_block_backward(self._h, _ptr(params), _ptr(grad_acc), _ptr(grads)))

    def sync(self) -> None:
        check(lib().dpb_sync(self._h))

    def profile(self, enable: bool) -> None:
        """Bracket every kernel launch with CUDA events (see dpb.h)."""
        check(lib().dpb_block_profile(self._h, int(enable)))

    def profile_read(self) -> dict:
        """{category: {launches, total_ms, bytes, flops, bytes_8d}} since profile(True);
        bytes with this build's fp32 storage, bytes_8d under SURVEY 8(d)'s model."""
        arr = (KernelStat * 32)()
        n = C.c_int()
        check(lib().dpb_block_profile_read(self._h, arr, 32, C.byref(n)))
        return {arr[i].name.decode(): {"launches": int(arr[i].launches), "total_ms": float(arr[i].total_ms),
                                       "bytes": float(arr[i].bytes), "flops": float(arr[i].flops),
                                       "bytes_8d": float(arr[i].bytes_8d)}
                for i in range(n.value)}

    def trace(self) -> dict:
        """OpTrace of the last forward + backward (dpb_block_trace): per-node
        {forward, backward, recompute} counts and per-kind FLOPs."""
        import numpy as np
        n = C.c_int()
        check(lib().dpb_block_trace(self._h, None, 0, None, C.byref(n)))
        counts = np.zeros(3 * n.value, dtype=np.int32)
        flops = np.zeros(21, dtype=np.float64)
        check(lib().dpb_block_trace(self._h, C.c_void_p(counts.ctypes.data), n.value,
                                    C.c_void_p(flops.ctypes.data), C.byref(n)))
        kinds = ["concat", "batchnorm", "relu", "conv", "pool", "linear", "loss"]
        f = flops.reshape(3, 7)
        return {"nodes": counts.reshape(-1, 3),
                "forward_flops": dict(zip(kinds, f[0])), "backward_flops": dict(zip(kinds, f[1])),
                "recompute_flops": dict(zip(kinds, f[2]))}

    # -- read-back in the reference layout -------------------------------------

    def feats(self) -> torch.Tensor:
        s = self.shape
        out = torch.empty((s.n, s.c_out, s.h, s.w), dtype=torch.float32, device=f"cuda:{self.device}")
        check(lib().dpb_block_read_feats(self._h, _ptr(out)))
        return out

    def z(self) -> torch.Tensor:
        s = self.shape
        out = torch.empty((s.m, s.n, s.bk, s.h, s.w), dtype=torch.float32, device=f"cuda:{self.device}")
        check(lib().dpb_block_read_z(self._h, _ptr(out)))
        return out

    def stats(self) -> torch.Tensor:
        out = torch.empty(self.shape.stat_elems, dtype=torch.float32, device=f"cuda:{self.device}")
        check(lib().dpb_block_read_stats(self._h, _ptr(out)))
        return out
