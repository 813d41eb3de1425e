"""Data-parallel plumbing.

The device path is native: `DpComm` wraps libdpb's NCCL communicator
(dpb_comm_*), and a `ModelPlan` with a communicator attached averages its
gradients inside `dpb_model_step`, one allreduce per block bucket issued on a
communication stream as each block's backward completes (`model_buckets`
lists them in issue order).  `GradientBuckets` is the same bucket schedule
over torch.distributed, used for the host-side (gloo) tests and for
dense-block-only runs.

The reference is single-device; its semantics are per-device batchnorm from
the current batch only. So a data-parallel step is: each rank
runs the full block forward+backward on its own shard of the global batch,
then the fp32 parameter gradients are summed over ranks and scaled by 1/P.
That is the gradient of the mean of the per-shard mean losses. BN running
statistics stay per rank.

`GradientBuckets` owns ONE flat fp32 buffer. Its per-block views are what the
blocks' backward writes (`BlockPlan.backward(..., grads=buckets.view(i))`), so
no concatenation is needed. Reduction is either:

* `reduce_all()`: one allreduce of the whole buffer after the step (bench.py:
  3 MB for BC-100, ~20 us over NVLink, cheaper than splitting the CUDA graph);
* `reduce_block(i)` + `finish()`: one async allreduce per block, issued as that
  block's backward completes (reverse block order). NCCL's stream is ordered
  after the compute stream at issue time, so the transfer overlaps the next
  block's backward ("buckets are issued per block").

Both paths run the same code under gloo (CPU tensors; tests/test_dp.py,
world size 2) and NCCL (CUDA tensors; bench.py under torchrun).
"""
from __future__ import annotations

from typing import Sequence

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist


def shard_range(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """Images [lo, hi) of the global batch that `rank` owns: contiguous, equal shards
    (rank r takes samples [B_r·r, B_r·(r+1)))."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if global_batch < world or global_batch % world:
        raise ValueError(f"global batch {global_batch} does not split evenly over {world} ranks")
    per = global_batch // world
    return rank * per, (rank + 1) * per


class GradientBuckets:
    """Flat fp32 gradient buffer with one bucket (view) per dense block."""

    def __init__(self, sizes: Sequence[int], device: torch.device | str = "cpu",
                 group: dist.ProcessGroup | None = None):
        if any(int(s) <= 0 for s in sizes):
            raise ValueError("every bucket needs at least one element")
        self.sizes = [int(s) for s in sizes]
        self.offsets = [0]
        for s in self.sizes:
            self.offsets.append(self.offsets[-1] + s)
        self.flat = torch.zeros(self.offsets[-1], dtype=torch.float32, device=device)
        self.group = group
        self._pending: list = []

    @property
    def world(self) -> int:
        return dist.get_world_size(self.group) if dist.is_initialized() else 1

    def view(self, i: int) -> torch.Tensor:
        return self.flat[self.offsets[i]:self.offsets[i + 1]]

    def reduce_block(self, i: int) -> None:
        """Start the allreduce of bucket i (async); call once block i's backward is enqueued."""
        if self.world == 1:
            return
        self._pending.append((i, dist.all_reduce(self.view(i), group=self.group, async_op=True)))

    def finish(self) -> torch.Tensor:
        """Wait for every started bucket, then scale by 1/P. Returns the flat buffer."""
        world = self.world
        for i, work in self._pending:
            work.wait()
            self.view(i).mul_(1.0 / world)
        self._pending.clear()
        return self.flat

    def reduce_all(self) -> torch.Tensor:
        """One allreduce of the whole buffer (sum), scaled by 1/P."""
        if self._pending:
            raise RuntimeError("reduce_all while per-block reductions are pending")
        world = self.world
        if world > 1:
            dist.all_reduce(self.flat, group=self.group)
            self.flat.mul_(1.0 / world)
        return self.flat


def model_buckets(cfg) -> list[tuple[int, int]]:
    """The whole-network gradient buckets [begin, end) in the order
    dpb_model_step reduces them (last block with the head first, ..., block 0
    with its transition and the stem last).  They tile [0, param_elems)."""
    from ._lib import check, lib
    from .model import model_desc
    d = model_desc(cfg, 1)
    out = np.zeros(2 * 16, dtype=np.int64)
    n = C.c_int()
    check(lib().dpb_model_buckets(C.byref(d), C.c_void_p(out.ctypes.data), 16, C.byref(n)))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n.value)]


class DpComm:
    """libdpb's NCCL communicator for this rank (dpb_comm_init).  Rank 0's
    unique id travels over the already-initialised torch.distributed group
    (any backend).  Attach with ModelPlan.set_comm."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        from ._lib import check, lib
        idb = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            check(lib().dpb_comm_unique_id(C.c_void_p(idb.ctypes.data)))
        if world > 1:
            t = torch.from_numpy(idb)
            if dist.get_backend(group) == "nccl":
                t = t.cuda(device)
            dist.broadcast(t, src=0, group=group)
            idb = t.cpu().numpy().copy()
        h = C.c_void_p()
        check(lib().dpb_comm_init(world, rank, C.c_void_p(idb.ctypes.data), device, C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world

    @property
    def handle(self):
        return self._h

    def check(self) -> None:
        from ._lib import check, lib
        check(lib().dpb_comm_check(self._h))

    def close(self) -> None:
        from ._lib import lib
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().dpb_comm_destroy(self._h)
            self._h = C.c_void_p()
