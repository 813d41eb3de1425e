"""Per-op device entry points mirroring denseplan::ops (ops.hpp:53-387).

Tensors are fp32 NCHW torch CUDA tensors; every call goes to libdpb.so.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import errors
from ._lib import check, lib
from .block import _ptr


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _out(out, shape, device):
    if out is None:
        return torch.empty(shape, device=device)
    if tuple(out.shape) != tuple(shape) or out.dtype != torch.float32 or not out.is_contiguous():
        raise errors.ShapeError(f"output buffer {tuple(out.shape)} does not match {tuple(shape)}")
    return out


def batch_statistics(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-channel mean and biased variance (ops.hpp:138-162)."""
    n, c, h, w = x.shape
    mean = torch.empty(c, device=x.device)
    var = torch.empty(c, device=x.device)
    check(lib().dpb_op_batch_statistics(_ptr(x), n, c, h, w, _ptr(mean), _ptr(var), _stream()))
    return mean, var


def batchnorm_apply(x, gamma, beta, mean, var, relu: bool = False) -> torch.Tensor:
    """gamma*(x-mean)*inv + beta (ops.hpp:115-134), optionally + relu."""
    n, c, h, w = x.shape
    out = torch.empty_like(x)
    check(lib().dpb_op_batchnorm_apply(_ptr(x), n, c, h, w, _ptr(gamma), _ptr(beta), _ptr(mean),
                                       _ptr(var), int(relu), _ptr(out), _stream()))
    return out


def batchnorm_backward(grad_y, x, gamma, mean, var, out=None):
    """Exact train-mode BN gradients (ops.hpp:206-243) -> (gx, dgamma, dbeta).
    `out`, if given, is a contiguous fp32 buffer of x's shape that receives gx."""
    n, c, h, w = x.shape
    if grad_y.shape != x.shape:
        raise errors.ShapeError("batchnorm_backward shape mismatch")
    gx = _out(out, x.shape, x.device)
    dg = torch.empty(c, device=x.device)
    db = torch.empty(c, device=x.device)
    check(lib().dpb_op_batchnorm_backward(_ptr(grad_y), _ptr(x), n, c, h, w, _ptr(gamma), _ptr(mean),
                                          _ptr(var), _ptr(gx), _ptr(dg), _ptr(db), _stream()))
    return gx, dg, db


def conv2d_forward(x, weights, padding: int) -> torch.Tensor:
    """Stride-1 cross-correlation (ops.hpp:315-342)."""
    n, cin, h, w = x.shape
    cout, wc, kh, kw = weights.shape
    if wc != cin:
        raise errors.ShapeError(f"conv input channels {cin} != weight in_channels {wc}")
    oh, ow = h + 2 * padding - kh + 1, w + 2 * padding - kw + 1
    if oh < 1 or ow < 1:
        raise errors.ShapeError("conv output collapses to zero size")
    out = torch.empty((n, cout, oh, ow), device=x.device)
    check(lib().dpb_op_conv2d_forward(_ptr(x), n, cin, h, w, _ptr(weights), cout, kh, padding,
                                      _ptr(out), _stream()))
    return out


def conv2d_backward(grad_y, x, weights, padding: int, need_grad_x: bool = True, out=None):
    """Exact gradients (ops.hpp:346-387) -> (grad_x or None, grad_w).
    `out`, if given, receives grad_x (contiguous fp32, x's shape)."""
    n, cin, h, w = x.shape
    cout, _, kh, _ = weights.shape
    gx = _out(out, x.shape, x.device) if need_grad_x else None
    gw = torch.empty_like(weights)
    check(lib().dpb_op_conv2d_backward(_ptr(grad_y), _ptr(x), n, cin, h, w, _ptr(weights), cout, kh,
                                       padding, _ptr(gx), _ptr(gw), _stream()))
    return gx, gw


# ---- optimizer (train.hpp:43-70, schedule.hpp:46-62) -----------------------------------
def sgd_step(params, grads, velocity, lr: float, momentum: float = 0.9, weight_decay: float = 1e-4,
             nesterov: bool = False, stream=None) -> None:
    """In-place momentum SGD over flat fp32 CUDA tensors (dpb_sgd_step)."""
    import ctypes as C
    n = params.numel()
    if grads.numel() != n or velocity.numel() != n:
        raise ValueError("params / grads / velocity sizes differ")
    s = None if stream is None else C.c_void_p(stream.cuda_stream)
    check(lib().dpb_sgd_step(C.c_void_p(params.data_ptr()), C.c_void_p(grads.data_ptr()),
                             C.c_void_p(velocity.data_ptr()), n, float(lr), float(momentum),
                             float(weight_decay), int(nesterov), s))


def lr_at(kind: str, base_lr: float, total_epochs: int, epoch: int, milestones=(), factor: float = 0.1,
          floor: float = 0.0) -> float:
    """Learning rate of `epoch` for a step ("step") or cosine ("cosine") schedule."""
    import ctypes as C
    arr = (C.c_int32 * max(1, len(milestones)))(*milestones)
    out = C.c_double()
    check(lib().dpb_lr_at({"step": 0, "cosine": 1}[kind], float(base_lr), int(total_epochs),
                          C.cast(arr, C.c_void_p), len(milestones), float(factor), float(floor), int(epoch),
                          C.byref(out)))
    return out.value


def concat_forward(inputs: list) -> torch.Tensor:
    """concat_forward (ops.hpp:53-88): NCHW inputs sharing (n, h, w) -> their
    channel concatenation (a new tensor)."""
    if not inputs:
        raise errors.ShapeError("concat of zero inputs")
    n, _, h, w = inputs[0].shape
    for t in inputs:
        if t.shape[0] != n or t.shape[2] != h or t.shape[3] != w:
            raise errors.ShapeError(f"concat input {tuple(t.shape)} incompatible")
    chans = [int(t.shape[1]) for t in inputs]
    dst = torch.empty((n, sum(chans), h, w), device=inputs[0].device)
    ptrs = (C.c_void_p * len(inputs))(*[t.data_ptr() for t in inputs])
    ch = (C.c_int64 * len(inputs))(*chans)
    check(lib().dpb_op_concat_forward(len(inputs), C.cast(ptrs, C.c_void_p), C.cast(ch, C.c_void_p), n, h, w,
                                      _ptr(dst), dst.shape[1], _stream()))
    return dst


def concat_backward(grad_out: torch.Tensor, splits: list) -> list:
    """concat_backward (ops.hpp:91-107): the gradient's channel slices as
    separate tensors (copies; the reference returns views)."""
    n, c, h, w = grad_out.shape
    outs = [torch.empty((n, int(s), h, w), device=grad_out.device) for s in splits]
    ptrs = (C.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
    ch = (C.c_int64 * max(1, len(outs)))(*[int(s) for s in splits])
    check(lib().dpb_op_concat_backward(_ptr(grad_out), n, c, h, w, len(outs), C.cast(ch, C.c_void_p),
                                       C.cast(ptrs, C.c_void_p), _stream()))
    return outs


def relu_forward(x: torch.Tensor, inplace: bool = False) -> torch.Tensor:
    """relu_forward / relu_inplace (ops.hpp:248-264)."""
    dst = x if inplace else torch.empty_like(x)
    check(lib().dpb_op_relu_forward(_ptr(x), x.numel(), _ptr(dst), _stream()))
    return dst


def relu_backward(grad_y: torch.Tensor, ref: torch.Tensor, inplace: bool = False) -> torch.Tensor:
    """relu_backward(_inplace) (ops.hpp:268-287): grad_y where ref > 0, else 0."""
    if grad_y.shape != ref.shape:
        raise errors.ShapeError("relu_backward shape mismatch")
    gx = grad_y if inplace else torch.empty_like(grad_y)
    check(lib().dpb_op_relu_backward(_ptr(grad_y), _ptr(ref), grad_y.numel(), _ptr(gx), _stream()))
    return gx
