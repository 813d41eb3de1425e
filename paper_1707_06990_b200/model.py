"""Host-side model arithmetic and configs (densenet.hpp / peak_model.hpp /
rng.hpp), computed by libdpb.so's host code.

``CONFIGS`` holds the five BASELINE.json configurations.  DenseNet-264 is
built as blocks (6, 12, 64, 48) — the 33M / 73M models BASELINE names — not
the reference's ``paper-264-*`` presets (6, 32, 64, 48).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib
from .block import BlockShape

STRATEGIES = {"naive": 0, "shared-grad": 1, "shared-all": 2}
ARENAS = ["params", "feature_owned", "shared1", "shared2", "shared_grad", "scratch"]


@dataclass(frozen=True)
class DenseNetConfig:
    """densenet.hpp:46-85 (pre-activation; bottleneck width 4k)."""
    block_sizes: tuple
    growth_rate: int
    bottleneck: bool = True
    compression: float = 0.5
    num_classes: int = 10
    initial_channels: int = -1
    in_shape: tuple = (3, 32, 32)   # (c, h, w) of the network input
    activation: str = "pre"         # "pre" | "post" (densenet.hpp ActivationOrder)
    # "3x3": the reference's conv 3x3/1 stem (graph.hpp:430); "imagenet": conv
    # 7x7/2 -> BN -> ReLU -> max-pool 3x3/2 (extension; 224 -> 56)
    stem: str = "3x3"

    @property
    def c0(self) -> int:
        return self.initial_channels if self.initial_channels > 0 else 2 * self.growth_rate

    def _args(self):
        arr = (C.c_int32 * len(self.block_sizes))(*self.block_sizes)
        return [len(self.block_sizes), C.cast(arr, C.c_void_p), self.growth_rate,
                int(self.bottleneck), float(self.compression), self.num_classes,
                self.c0], arr

    @property
    def stem_id(self) -> int:
        return {"3x3": 0, "imagenet": 1}[self.stem]

    def stem_out_hw(self) -> tuple:
        """Spatial size entering block 0: the reference's 3x3/1 stem keeps it
        (graph.hpp:430); the ImageNet stem is conv 7x7/2 pad 3 then max-pool
        3x3/2 pad 1 ((in + 2p - k) / s + 1 twice, ops.hpp:292-294)."""
        _, h, w = self.in_shape
        if self.stem == "imagenet":
            h, w = ((h - 1) // 2 + 1 - 1) // 2 + 1, ((w - 1) // 2 + 1 - 1) // 2 + 1
        return h, w

    def block_shapes(self, batch: int) -> list[BlockShape]:
        """Per-block geometry (net_geometry, densenet.hpp:141-180) after the stem."""
        h, w = self.stem_out_hw()
        c = self.c0
        out = []
        for b, m in enumerate(self.block_sizes):
            out.append(BlockShape(batch, h, w, c, m, self.growth_rate, 4 * self.growth_rate))
            c = c + m * self.growth_rate
            if b + 1 < len(self.block_sizes):
                c = int(np.floor(self.compression * c))
                h, w = (h - 2) // 2 + 1, (w - 2) // 2 + 1
        return out


def count_parameters(cfg: DenseNetConfig, in_c: int = 3) -> int:
    """densenet.hpp:234-275."""
    args, keep = cfg._args()
    out = C.c_int64()
    check(lib().dpb_count_parameters(*args, in_c, C.byref(out)))
    return out.value


def predict_peak_elements(cfg: DenseNetConfig, strategy: str, batch: int, in_c: int, in_h: int,
                          in_w: int) -> dict:
    """peak_model.hpp:37-158, per arena element counts."""
    args, keep = cfg._args()
    out = np.zeros(6, dtype=np.int64)
    check(lib().dpb_predict_peak_elements(*args, STRATEGIES[strategy], batch, in_c, in_h, in_w,
                                          C.c_void_p(out.ctypes.data)))
    return dict(zip(ARENAS, (int(v) for v in out)))


def rng_normal(seed: int, count: int) -> np.ndarray:
    """Rng(seed).normal() draws (rng.hpp:36-49), as float32."""
    out = np.empty(count, dtype=np.float32)
    check(lib().dpb_rng_fill_normal(seed, C.c_void_p(out.ctypes.data), count))
    return out


# BASELINE.json configs.  The ImageNet configs use the
# 7x7/2 + max-pool stem at 224x224; their "@56" twins are the reference's own
# geometry for the same networks (3x3/1 stem on a 3x56x56 input: identical
# dense blocks, transitions and head — what GraphPlan can run).
CONFIGS = {
    "cfg1": DenseNetConfig((12,), 12, True, 1.0, 10, 24, (3, 32, 32)),
    "bc100": DenseNetConfig((16, 16, 16), 12, True, 0.5, 10, 24, (3, 32, 32)),
    "d121": DenseNetConfig((6, 12, 24, 16), 32, True, 0.5, 1000, 64, (3, 224, 224), stem="imagenet"),
    "d264k32": DenseNetConfig((6, 12, 64, 48), 32, True, 0.5, 1000, 64, (3, 224, 224), stem="imagenet"),
    "d264k48": DenseNetConfig((6, 12, 64, 48), 48, True, 0.5, 1000, 96, (3, 224, 224), stem="imagenet"),
    "d121@56": DenseNetConfig((6, 12, 24, 16), 32, True, 0.5, 1000, 64, (3, 56, 56)),
    "d264k32@56": DenseNetConfig((6, 12, 64, 48), 32, True, 0.5, 1000, 64, (3, 56, 56)),
    "d264k48@56": DenseNetConfig((6, 12, 64, 48), 48, True, 0.5, 1000, 96, (3, 56, 56)),
}


def param_segments(cfg: DenseNetConfig) -> list[tuple[str, int, int]]:
    """(name, elements, fan_in) of every parameter tensor in registration
    order; fan_in 0 marks BN gamma (1) / beta and the linear bias (0)."""
    k, bk, in_c = cfg.growth_rate, 4 * cfg.growth_rate, cfg.in_shape[0]
    if cfg.stem == "imagenet":
        segs = [("stem.conv.w", cfg.c0 * in_c * 49, in_c * 49), ("stem.bn.gamma", cfg.c0, 0),
                ("stem.bn.beta", cfg.c0, 0)]
    else:
        segs = [("stem.conv.w", cfg.c0 * in_c * 9, in_c * 9)]
    shapes = cfg.block_shapes(1)
    for b, shp in enumerate(shapes):
        for l in range(shp.m):
            c = shp.c_in(l)
            segs += [(f"b{b}.l{l}.bn_a.gamma", c, 0), (f"b{b}.l{l}.bn_a.beta", c, 0),
                     (f"b{b}.l{l}.conv_a.w", bk * c, c), (f"b{b}.l{l}.bn_b.gamma", bk, 0),
                     (f"b{b}.l{l}.bn_b.beta", bk, 0), (f"b{b}.l{l}.conv_b.w", k * bk * 9, bk * 9)]
        C_ = shp.c_out
        if b + 1 < len(shapes):
            cout = int(np.floor(cfg.compression * C_))
            segs += [(f"t{b}.bn.gamma", C_, 0), (f"t{b}.bn.beta", C_, 0), (f"t{b}.conv.w", cout * C_, C_)]
        else:
            segs += [("head.bn.gamma", C_, 0), ("head.bn.beta", C_, 0),
                     ("head.linear.w", cfg.num_classes * C_, -C_), ("head.linear.b", cfg.num_classes, 0)]
    return segs

def param_shapes(cfg: DenseNetConfig) -> list[tuple[str, tuple]]:
    """(registered name, (n, c, h, w)) of every parameter (graph.hpp:351-390,
    :430-600), in registration order."""
    k, bk, in_c = cfg.growth_rate, 4 * cfg.growth_rate, cfg.in_shape[0]
    out = []
    for name, n, fan in param_segments(cfg):
        if name == "stem.conv.w":
            kk = 7 if cfg.stem == "imagenet" else 3
            shape = (cfg.c0, in_c, kk, kk)
        elif name.endswith(".conv_b.w"):
            shape = (k, bk, 3, 3)
        elif name.endswith(".conv_a.w"):
            shape = (bk, n // bk, 1, 1)
        elif name.endswith(".conv.w"):
            shape = (n // fan, fan, 1, 1)
        elif name == "head.linear.w":
            shape = (cfg.num_classes, n // cfg.num_classes, 1, 1)
        else:  # bn gamma / beta, linear bias
            shape = (1, n, 1, 1)
        assert int(np.prod(shape)) == n, name
        out.append((name, shape))
    return out

def _ckpt_tables(cfg: DenseNetConfig, with_velocity: bool):
    entries = param_shapes(cfg)
    if with_velocity:
        entries = entries + [("velocity." + n, s) for n, s in entries]
    names = (C.c_char_p * len(entries))(*[n.encode() for n, _ in entries])
    dims = np.array([s for _, s in entries], dtype=np.int64).reshape(-1)
    return entries, names, dims

def save_checkpoint(cfg: DenseNetConfig, path: str, params, velocity=None, epoch: int = 0) -> None:
    """DPLN checkpoint of the parameters (+ SGD velocities as a training
    checkpoint, train.hpp:149-172); device or host tensors."""
    import torch
    entries, names, dims = _ckpt_tables(cfg, velocity is not None)
    data = params.detach().float().cpu()
    if velocity is not None:
        data = torch.cat([data, velocity.detach().float().cpu()])
    data = np.ascontiguousarray(data.numpy())
    check(lib().dpb_checkpoint_save(path.encode(), len(entries), C.cast(names, C.c_void_p),
                                    dims.ctypes.data, data.ctypes.data, int(epoch)))

def load_checkpoint(cfg: DenseNetConfig, path: str, with_velocity: bool = False):
    """Returns (params, velocity or None, epoch) as host fp32 tensors."""
    import torch
    entries, names, dims = _ckpt_tables(cfg, with_velocity)
    pe = sum(n for _, n, _ in param_segments(cfg))
    n = pe * (2 if with_velocity else 1)
    data = np.zeros(n, dtype=np.float32)
    ep = C.c_int()
    check(lib().dpb_checkpoint_load(path.encode(), len(entries), C.cast(names, C.c_void_p),
                                    dims.ctypes.data, data.ctypes.data, C.byref(ep)))
    t = torch.from_numpy(data)
    if with_velocity:
        return t[:pe].clone(), t[pe:].clone(), ep.value
    return t, None, ep.value


def model_desc(cfg: DenseNetConfig, batch: int, dtype: str = "fp32"):
    """The dpb_model_desc of `cfg` (include/dpb.h)."""
    from ._lib import ModelDesc
    d = ModelDesc()
    d.nblocks = len(cfg.block_sizes)
    for i, m in enumerate(cfg.block_sizes):
        d.blocks[i] = m
    d.k = cfg.growth_rate
    d.compression = float(cfg.compression)
    d.classes = cfg.num_classes
    d.c0 = cfg.c0
    d.in_c, d.in_h, d.in_w = cfg.in_shape
    d.batch = batch
    d.dtype = {"fp32": 0, "bf16": 1}[dtype]
    d.stem = cfg.stem_id
    return d


def model_sizes(cfg: DenseNetConfig) -> tuple:
    """(param_elems, running_elems) of the whole network (dpb_model_sizes)."""
    d = model_desc(cfg, 1)
    pe, re_ = C.c_int64(), C.c_int64()
    check(lib().dpb_model_sizes(C.byref(d), C.byref(pe), C.byref(re_)))
    return pe.value, re_.value


def init_params(cfg: DenseNetConfig, seed: int) -> np.ndarray:
    """GraphPlan::build's parameters for `seed` in registration order, replayed
    draw for draw on the host by libdpb (dpb_model_init_params; graph.hpp:
    351-390, :405-600, rng.hpp:36-49): bit-identical to the reference's
    params() for the 3x3 stem."""
    d = model_desc(cfg, 1)
    out = np.empty(model_sizes(cfg)[0], dtype=np.float32)
    check(lib().dpb_model_init_params(C.byref(d), int(seed), C.c_void_p(out.ctypes.data)))
    return out


class ModelPlan:
    """Whole-network training step on the GPU (``dpb_model_*``): the stem,
    dense blocks, transitions, head and softmax cross-entropy of
    GraphPlan<T>::forward / compute_loss / backward (graph.hpp:731-826,
    :1065-1183).  Parameters and gradients are flat in the reference's
    registration order (include/dpb.h)."""

    def __init__(self, cfg: DenseNetConfig, batch: int, dtype: str = "fp32", device: int | None = None,
                 stream=None):
        import torch

        self.cfg = cfg
        self.batch = batch
        d = model_desc(cfg, batch, dtype)
        if not cfg.bottleneck or cfg.activation != "pre":
            from .errors import ConfigError
            raise ConfigError("ModelPlan implements pre-activation bottleneck (DenseNet-B/BC) networks only")
        self._desc = d
        pe, re_ = C.c_int64(), C.c_int64()
        check(lib().dpb_model_sizes(C.byref(d), C.byref(pe), C.byref(re_)))
        self.param_elems, self.running_elems = pe.value, re_.value
        self.device = torch.cuda.current_device() if device is None else device
        h = C.c_void_p()
        s = None if stream is None else C.c_void_p(stream.cuda_stream)
        check(lib().dpb_model_create(C.byref(d), self.device, s, C.byref(h)))
        self._h = h

    def param_segments(self) -> list[tuple[str, int, int]]:
        return param_segments(self.cfg)

    def param_shapes(self) -> list[tuple[str, tuple]]:
        return param_shapes(self.cfg)

    def save_checkpoint(self, path: str, params, velocity=None, epoch: int = 0) -> None:
        save_checkpoint(self.cfg, path, params, velocity, epoch)

    def load_checkpoint(self, path: str, with_velocity: bool = False):
        return load_checkpoint(self.cfg, path, with_velocity)

    def init_params(self, seed: int = 0, device="cuda"):
        """GraphPlan::build's parameters for `seed`, replayed draw for draw by
        libdpb (dpb_model_init_params; graph.hpp:351-390, :405-600, rng.hpp):
        bit-identical to the reference's params() for the 3x3 stem."""
        import torch
        return torch.from_numpy(init_params(self.cfg, seed)).to(device)

    def initial_running(self, device="cuda"):
        """Running means 0 / variances 1 in the model's running layout."""
        import torch
        parts = []
        if self.cfg.stem == "imagenet":  # stem BN
            parts.append(torch.cat([torch.zeros(self.cfg.c0), torch.ones(self.cfg.c0)]))
        shapes = self.cfg.block_shapes(self.batch)
        for b, shp in enumerate(shapes):
            parts.append(shp.initial_running("cpu"))
            C_ = shp.c_out
            parts.append(torch.cat([torch.zeros(C_), torch.ones(C_)]))  # transition b or head
        return torch.cat(parts).to(device)

    def step(self, x, labels, params, running, grads, loss) -> None:
        """x NCHW fp32, labels int32 [batch], params / grads flat fp32, running
        flat fp32 (updated), loss a 1-element fp32 device tensor."""
        def ptr(t):
            return C.c_void_p(t.data_ptr())
        check(lib().dpb_model_step(self._h, ptr(x), ptr(labels), ptr(params), ptr(running), ptr(grads),
                                   ptr(loss)))

    def sync(self) -> None:
        check(lib().dpb_model_sync(self._h))

    def wait_input(self, stream) -> None:
        """Make `stream` (a torch.cuda.Stream) wait until the last enqueued step
        has read its input images and labels (dpb_model_wait_input): the next
        batch's host-to-device copy may then overwrite them while that step
        finishes."""
        check(lib().dpb_model_wait_input(self._h, C.c_void_p(stream.cuda_stream)))

    def set_comm(self, comm) -> None:
        """Attach a dp.DpComm (or None): dpb_model_step then averages the
        gradients over the ranks, bucket by bucket, overlapped with backward."""
        check(lib().dpb_model_set_comm(self._h, None if comm is None else comm.handle))
        self._comm = comm  # keep the communicator alive while attached

    def launch_count(self) -> int:
        """Kernels one training step launches (the captured graph's kernel nodes)."""
        return int(lib().dpb_model_launch_count(self._h))

    def memory(self) -> dict:
        """libdpb's device-memory accounting of the whole step (dpb_model_memory_stats,
        MemoryStats of alloctrace.hpp): bytes per arena, the combined feature
        (activation) peak and the total allocated."""
        from ._lib import MemoryStats
        st = MemoryStats()
        check(lib().dpb_model_memory_stats(self._h, C.byref(st)))
        by = {name: int(st.peak_bytes[i]) for i, name in enumerate(ARENAS)}
        return {"by_arena": by, "activation_bytes": int(st.total_feature_peak_bytes),
                "total_bytes": sum(by.values())}

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().dpb_model_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
