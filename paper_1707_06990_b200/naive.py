"""Naive and SharedGradient dense blocks on the GPU.

These are the reference's two store-everything execution strategies
(ExecutionStrategy::Naive / ::SharedGradient, graph.hpp:273-310).  The peak
model (peak_model.hpp:57-90, 139-146) accounts for them per pre-activation
bottleneck layer with c input channels (x N*H*W elements):

    cat    the concatenation copy                    c
    bn     BN_a+ReLU output c, BN_b+ReLU output bk   c + bk
    owned  z (bk) and y (k)                          bk + k
    grad   transients g_b, g_z (bk), g_a, g_cat (c)  2bk + 2c

Per block, cat also holds the block-output concatenation (C) and grad holds
the block accumulator (C).  Under Naive every gradient transient lives until
the end of the step.  Under SharedGradient they come from one gradient region
of four slots, each sized to the largest transient or accumulator: two
accumulators that overlap at the block handoff, and two transient slots.

`NaiveBlock` runs either strategy with the unfused per-op kernels of the C ABI
(`ops.batch_statistics / batchnorm_apply / batchnorm_backward / conv2d_*`,
fp32 NCHW).  It materialises each of these tensors, so the footprint is a
device measurement: `accounting()` sums the live storage per arena, and
tests/test_naive_gpu.py checks it against `predict_peak_elements`.  It is the
memory and speed baseline of the memory-efficient path (`BlockPlan`), not a
product path.  Flat parameters and gradients use the dpb_block layout
(block.py BlockShape.param_offsets).  The ReLU masks and the concatenation
copies are plain device elementwise / copy ops.
"""
from __future__ import annotations

import torch

from . import ops
from .block import BlockShape

STRATEGIES = ("naive", "shared-gradient")


class NaiveBlock:
    def __init__(self, shape: BlockShape, strategy: str = "naive", device="cuda"):
        if strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
        self.s = shape
        self.strategy = strategy
        self.device = device
        self.saved: list[dict] = []
        self.out_cat = None
        self.keep: list[torch.Tensor] = []   # Naive: every gradient transient of the step
        self.acc = None                      # Naive: the block accumulator
        self.region = None                   # SharedGradient: [4, slot] gradient region
        if strategy == "shared-gradient":
            s = shape
            slot = max(s.bk, s.c_in(s.m - 1), s.c_out) * s.pixels
            self.region = torch.empty((4, slot), device=device)

    def _slot(self, i: int, shape) -> torch.Tensor:
        n = 1
        for d in shape:
            n *= d
        return self.region[i, :n].view(shape)

    def _layer_params(self, params, l):
        s = self.s
        c = s.c_in(l)
        o = s.param_offsets()[l]
        ga, ba = params[o:o + c], params[o + c:o + 2 * c]
        w1 = params[o + 2 * c:o + 2 * c + s.bk * c].view(s.bk, c, 1, 1)
        o2 = o + 2 * c + s.bk * c
        gb, bb = params[o2:o2 + s.bk], params[o2 + s.bk:o2 + 2 * s.bk]
        w2 = params[o2 + 2 * s.bk:o2 + 2 * s.bk + 9 * s.k * s.bk].view(s.k, s.bk, 3, 3)
        return ga, ba, w1, gb, bb, w2

    def forward(self, x_in: torch.Tensor, params: torch.Tensor) -> torch.Tensor:
        """x_in NCHW [n, c0, h, w]; returns the block-output concatenation."""
        s = self.s
        feats = [x_in]
        self.saved = []
        for l in range(s.m):
            ga, ba, w1, gb, bb, w2 = self._layer_params(params, l)
            cat = torch.cat(feats, dim=1)                             # cat (c)
            ma, va = ops.batch_statistics(cat)
            a = ops.batchnorm_apply(cat, ga, ba, ma, va, relu=True)   # bn (c)
            z = ops.conv2d_forward(a, w1, 0)                          # owned (bk)
            mb, vb = ops.batch_statistics(z)
            b = ops.batchnorm_apply(z, gb, bb, mb, vb, relu=True)     # bn (bk)
            y = ops.conv2d_forward(b, w2, 1)                          # owned (k)
            self.saved.append(dict(cat=cat, a=a, z=z, b=b, y=y, ma=ma, va=va, mb=mb, vb=vb))
            feats.append(y)
        self.out_cat = torch.cat(feats, dim=1)                        # cat (C)
        return self.out_cat

    def backward(self, params: torch.Tensor, grad_acc: torch.Tensor, grads: torch.Tensor) -> torch.Tensor:
        """grad_acc NCHW [n, C, h, w]: the block-output gradient, accumulated in
        place like dpb_block_backward (graph.hpp backward walk).  grads is flat,
        in the dpb_block layout."""
        s = self.s
        shared = self.strategy == "shared-gradient"
        # the accumulator: slot 0 of the region, or a tensor of its own kept to step end
        acc = self._slot(0, grad_acc.shape) if shared else torch.empty_like(grad_acc)
        acc.copy_(grad_acc)
        self.acc = None if shared else acc
        self.keep = []
        n, h, w = s.n, s.h, s.w
        for l in reversed(range(s.m)):
            ga, ba, w1, gb, bb, w2 = self._layer_params(params, l)
            sv = self.saved[l]
            c = s.c_in(l)
            g_y = acc[:, c:c + s.k].contiguous()
            tb = self._slot(2, (n, s.bk, h, w)) if shared else None
            g_b, dw2 = ops.conv2d_backward(g_y, sv["b"], w2, 1, out=tb)            # grad (bk)
            g_b.masked_fill_(sv["b"] <= 0, 0.0)
            tz = self._slot(3, (n, s.bk, h, w)) if shared else None
            g_z, dgb, dbb = ops.batchnorm_backward(g_b, sv["z"], gb, sv["mb"], sv["vb"], out=tz)  # (bk)
            ta = self._slot(2, (n, c, h, w)) if shared else None
            g_a, dw1 = ops.conv2d_backward(g_z, sv["a"], w1, 0, out=ta)            # grad (c)
            g_a.masked_fill_(sv["a"] <= 0, 0.0)
            tc = self._slot(3, (n, c, h, w)) if shared else None
            g_cat, dga, dba = ops.batchnorm_backward(g_a, sv["cat"], ga, sv["ma"], sv["va"], out=tc)  # (c)
            acc[:, :c] += g_cat
            if not shared:
                self.keep += [g_b, g_z, g_a, g_cat]
            o = s.param_offsets()[l]
            o2 = o + 2 * c + s.bk * c
            grads[o:o + c] = dga
            grads[o + c:o + 2 * c] = dba
            grads[o + 2 * c:o2] = dw1.reshape(-1)
            grads[o2:o2 + s.bk] = dgb
            grads[o2 + s.bk:o2 + 2 * s.bk] = dbb
            grads[o2 + 2 * s.bk:o2 + 2 * s.bk + 9 * s.k * s.bk] = dw2.reshape(-1)
        grad_acc.copy_(acc)
        return grad_acc

    def accounting(self) -> dict:
        """Elements held at the end of the step, per arena, counted from the live
        storage (peak_model.hpp:139-146 arena split): cat, bn, owned, and grad
        (Naive: every transient plus the accumulator; SharedGradient: the
        four-slot region)."""
        cat = sum(sv["cat"].numel() for sv in self.saved) + self.out_cat.numel()
        bn = sum(sv["a"].numel() + sv["b"].numel() for sv in self.saved)
        owned = sum(sv["z"].numel() + sv["y"].numel() for sv in self.saved)
        if self.strategy == "naive":
            grad = sum(t.numel() for t in self.keep) + (self.acc.numel() if self.acc is not None else 0)
        else:
            grad = self.region.numel()
        return {"cat": cat, "bn": bn, "owned": owned, "grad": grad}

    def retained_bytes(self) -> int:
        return 4 * sum(self.accounting().values())


def naive_network_replay(cfg, batch: int, device="cuda") -> dict:
    """The whole network under the reference's Naive strategy (graph.hpp:
    279-310: every forward tensor and every gradient transient held until the
    step ends), measured with the CUDA caching allocator's high-water mark.

    The dense blocks run for real through `NaiveBlock` (unfused per-op
    kernels, fp32), one after another, keeping their state, then backward in
    reverse.  The stem, transition and head tensors the strategy would hold
    (peak_model.hpp:57-133: conv / BN / pool outputs, their gradient
    transients) are allocated at their shapes without being computed — they
    are small next to the blocks.  Parameters and parameter gradients are
    allocated before the baseline (peak_model counts them under Params).
    Returns bytes: allocator peak, and the reference peak model's Naive
    feature arenas for the same network, fp32."""
    from .model import predict_peak_elements
    dev = torch.device(device)
    shapes = cfg.block_shapes(batch)
    g = torch.Generator(device="cpu").manual_seed(11)
    params = [(torch.randn(s.param_elems, generator=g) * 0.05 + 0.5).to(dev) for s in shapes]
    grads = [torch.empty(s.param_elems, device=dev) for s in shapes]
    torch.cuda.synchronize(dev)
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hold = []
    N, c0 = batch, cfg.c0
    _, h, w = cfg.in_shape
    if cfg.stem == "imagenet":
        h1, w1 = (h - 1) // 2 + 1, (w - 1) // 2 + 1
        hold += [torch.empty((N, c0, h1, w1), device=dev) for _ in range(2)]   # conv out, BN+ReLU out
    else:
        hold.append(torch.empty((N, c0, h, w), device=dev))                   # stem conv out
    x = torch.randn((N, c0, shapes[0].h, shapes[0].w), device=dev)            # block-0 input (pool out)
    blocks = []
    for b, s in enumerate(shapes):
        nb = NaiveBlock(s, "naive", dev)
        nb.forward(x, params[b])
        blocks.append(nb)
        C = s.c_out
        if b + 1 < len(shapes):  # transition: BN+ReLU out, conv out, pooled out
            cout = shapes[b + 1].c0
            hold += [torch.empty((N, C, s.h, s.w), device=dev), torch.empty((N, cout, s.h, s.w), device=dev)]
            x = torch.randn((N, cout, shapes[b + 1].h, shapes[b + 1].w), device=dev)
        else:                    # head: BN+ReLU out, pooled features, logits
            hold += [torch.empty((N, C, s.h, s.w), device=dev), torch.empty((N, C), device=dev),
                     torch.empty((N, cfg.num_classes), device=dev)]
    for b in reversed(range(len(shapes))):
        s = shapes[b]
        C = s.c_out
        if b + 1 == len(shapes):  # head backward transients: d(gap), d(act)
            hold += [torch.empty((N, C), device=dev), torch.empty((N, C, s.h, s.w), device=dev)]
        acc = torch.randn((N, C, s.h, s.w), device=dev)   # the block accumulator the consumer's BN bwd writes
        hold.append(acc)
        blocks[b].backward(params[b], acc, grads[b])
        if b > 0:                 # transition b-1 backward transients: d(conv out), d(BN in)
            p = shapes[b - 1]
            hold += [torch.empty((N, s.c0, p.h, p.w), device=dev), torch.empty((N, p.c_out, p.h, p.w), device=dev)]
    e1.record()
    torch.cuda.synchronize(dev)
    peak = torch.cuda.max_memory_allocated(dev) - base
    # the reference's geometry: its 3x3/1 stem at the block-0 field
    pred = predict_peak_elements(cfg, "naive", batch, cfg.in_shape[0], shapes[0].h, shapes[0].w)
    out = {"allocator_peak_bytes": int(peak),
           "reference_peak_model_bytes": 4 * sum(v for k, v in pred.items() if k != "params"),
           "blocks_ms": e0.elapsed_time(e1),
           "note": ("reference Naive strategy, fp32: dense blocks computed by NaiveBlock (unfused per-op "
                    "kernels), stem / transition / head tensors allocated at their shapes; CUDA caching "
                    "allocator high-water above the parameters.  The peak model uses the reference's "
                    "3x3/1 stem geometry; NaiveBlock keeps one extra accumulator copy per block")}
    del blocks, hold
    torch.cuda.empty_cache()
    return out
