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

    @property
    def c0(self) -> int:
        return self.initial_channels if self.initial_channels > 0 else 2 * self.growth_rate

    def _args(self):
        arr = (C.c_int32 * len(self.block_sizes))(*self.block_sizes)
        return [len(self.block_sizes), C.cast(arr, C.c_void_p), self.growth_rate,
                int(self.bottleneck), float(self.compression), self.num_classes,
                self.c0], arr

    def block_shapes(self, batch: int, stem_stride: int = 1) -> list[BlockShape]:
        """Per-block geometry (net_geometry, densenet.hpp:141-180).  The
        reference stem is 3x3 stride 1 (graph.hpp:430); ``stem_stride`` 4
        reproduces the ImageNet 7x7/2 + max-pool geometry."""
        _, h, w = self.in_shape
        h, w = h // stem_stride, w // stem_stride
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


# BASELINE.json configs
CONFIGS = {
    "cfg1": DenseNetConfig((12,), 12, True, 1.0, 10, 24, (3, 32, 32)),
    "bc100": DenseNetConfig((16, 16, 16), 12, True, 0.5, 10, 24, (3, 32, 32)),
    "d121": DenseNetConfig((6, 12, 24, 16), 32, True, 0.5, 1000, 64, (3, 224, 224)),
    "d264k32": DenseNetConfig((6, 12, 64, 48), 32, True, 0.5, 1000, 64, (3, 224, 224)),
    "d264k48": DenseNetConfig((6, 12, 64, 48), 48, True, 0.5, 1000, 96, (3, 224, 224)),
}
