"""Training step of a chain of dense blocks fed from host (pinned) buffers.

`HostBlockChain` is the end-to-end entry point the bench's `e2e` number uses:
every step copies each block's input features and upstream gradient from
pinned host memory, runs the block forwards and the block backwards in reverse
order (`BlockPlan`, the C ABI), optionally all-reduces the gradients
(`GradientBuckets`), and copies the flat fp32 parameter gradients back to
pinned host memory.

Host->device copies run on their own stream and are ordered per block with
events: block b's forward waits only for its own input, and its backward
waits only for its own upstream gradient. Copies for later blocks therefore
overlap the compute of earlier ones. A buffer is overwritten by the next
step's copy only after the kernels that read it have finished
(`dp/graph.hpp` has no host staging; this replaces the caller's own copies
around `GraphPlan::forward/backward`).
"""
from __future__ import annotations

from typing import Sequence

import torch

from .block import BlockPlan, BlockShape
from .dp import GradientBuckets


class HostBlockChain:
    def __init__(self, shapes: Sequence[BlockShape], params: Sequence[torch.Tensor],
                 running: Sequence[torch.Tensor], dtype: str = "bf16", layout: str = "nchw",
                 device: torch.device | None = None, stream: torch.cuda.Stream | None = None,
                 group=None):
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.current_stream(self.device)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.shapes = list(shapes)
        self.params = list(params)
        self.running = list(running)
        self.layout = layout
        self.plans = [BlockPlan(s, dtype=dtype, layout=layout, device=self.device.index, stream=self.stream)
                      for s in self.shapes]
        self.buckets = GradientBuckets([s.param_elems for s in self.shapes], device=self.device, group=group)
        self.grads_host = torch.empty(self.buckets.flat.numel(), pin_memory=True)

        def dev_buf(s: BlockShape, c: int) -> torch.Tensor:
            shape = (s.n, c, s.h, s.w) if layout == "nchw" else (s.n, s.h, s.w, c)
            return torch.empty(shape, device=self.device)

        self.x = [dev_buf(s, s.c0) for s in self.shapes]
        self.acc = [dev_buf(s, s.c_out) for s in self.shapes]
        ev = lambda: [torch.cuda.Event() for _ in self.shapes]  # noqa: E731
        self.x_ready, self.g_ready, self.fwd_done, self.bwd_done = ev(), ev(), ev(), ev()
        self._first = True

    def h2d_bytes(self) -> int:
        return sum(t.numel() * 4 for t in self.x) + sum(t.numel() * 4 for t in self.acc)

    def d2h_bytes(self) -> int:
        return self.grads_host.numel() * 4

    def step(self, x_host: Sequence[torch.Tensor], grad_host: Sequence[torch.Tensor]) -> torch.Tensor:
        """One forward+backward of every block from host inputs; returns the pinned host
        gradient buffer (valid once `self.stream` has been synchronised)."""
        nb = len(self.plans)
        cs, st = self.copy_stream, self.stream
        with torch.cuda.stream(cs):
            for b in range(nb):
                if not self._first:
                    cs.wait_event(self.fwd_done[b])    # previous step's forward read x[b]
                self.x[b].copy_(x_host[b], non_blocking=True)
                self.x_ready[b].record(cs)
            for b in reversed(range(nb)):
                if not self._first:
                    cs.wait_event(self.bwd_done[b])    # previous step's backward used acc[b]
                self.acc[b].copy_(grad_host[b], non_blocking=True)
                self.g_ready[b].record(cs)
        self._first = False
        with torch.cuda.stream(st):
            for b in range(nb):
                st.wait_event(self.x_ready[b])
                self.plans[b].forward(self.x[b], self.params[b], self.running[b], True)
                self.fwd_done[b].record(st)
            for b in reversed(range(nb)):
                st.wait_event(self.g_ready[b])
                self.plans[b].backward(self.params[b], self.acc[b], self.buckets.view(b))
                self.bwd_done[b].record(st)
            if self.buckets.world > 1:
                self.buckets.reduce_all()
            self.grads_host.copy_(self.buckets.flat, non_blocking=True)
        return self.grads_host

    def close(self) -> None:
        for p in self.plans:
            p.close()
