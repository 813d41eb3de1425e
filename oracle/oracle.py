"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes front end for the parity oracle (``_build/liboracle.so``, the plain-C
restatement in dp_oracle.c) and, when built, the reference itself
(``_ref/libdenseplan_ref.so``, the unmodified reference headers compiled by
oracle/Makefile).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline / reference legs may import this module; the product package
never does.

Array conventions match the reference (NCHW) and the flat per-block layouts
documented in dp_oracle.c:

* params / grads, per layer l (c = c0 + l*k):
  ``gamma_a[c] beta_a[c] W1[bk,c] gamma_b[bk] beta_b[bk] W2[k,bk,3,3]``
* stats / running, per layer: ``mean_a[c] var_a[c] mean_b[bk] var_b[bk]``
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdenseplan_ref.so")
REF_FAST_SO = os.path.join(HERE, "_ref", "libdenseplan_ref_fast.so")

_P = C.c_void_p
_I64 = C.c_int64


def build(ref: bool | None = None) -> None:
    """Build liboracle.so (always) and _ref (when /root/reference exists)."""
    targets = ["_build/liboracle.so"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/include")
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_P)


_lib = None
_ref = {}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _lib = C.CDLL(ORACLE_SO)
        for suf in ("f32", "f64"):
            f = getattr(_lib, f"dpo_block_forward_{suf}")
            f.restype = C.c_int
            f.argtypes = [_I64] * 7 + [_P] * 5 + [C.c_int]
            f = getattr(_lib, f"dpo_block_backward_{suf}")
            f.restype = C.c_int
            f.argtypes = [_I64] * 7 + [_P] * 6
        _lib.dpo_fill_normal_f64.argtypes = [C.c_uint64, _P, _I64]
        _lib.dpo_fill_normal_f32.argtypes = [C.c_uint64, _P, _I64]
        _lib.dpo_rng_u64_fill.argtypes = [C.c_uint64, _P, _I64]
    return _lib


def ref_lib(fast: bool = False):
    """The reference itself (oracle/_ref).  Raises if it was not built."""
    path = REF_FAST_SO if fast else REF_SO
    if path not in _ref:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference; run make -C oracle ref)")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        for suf in ("f32", "f64"):
            f = getattr(L, f"ref_block_harness_{suf}")
            f.restype = C.c_int
            f.argtypes = [_I64] * 7 + [_P, _P, _P, C.c_int] + [_P] * 5
            f = getattr(L, f"ref_check_block_harness_{suf}")
            f.restype = C.c_int
            f.argtypes = [C.c_int] * 6 + [C.c_uint64]
        cfg = [C.c_int, _P, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]
        L.ref_block_params_f32.restype = C.c_int
        L.ref_block_params_f32.argtypes = cfg + [C.c_int] * 3 + [_I64, C.c_uint64, C.c_int, _P]
        L.ref_model_step_f32.restype = C.c_int
        L.ref_model_step_f32.argtypes = cfg + [C.c_int] * 3 + [_I64, C.c_uint64, C.c_int, _P, _P, _P]
        L.ref_model_params_f32.restype = C.c_int
        L.ref_model_params_f32.argtypes = cfg + [C.c_int] * 3 + [_I64, C.c_uint64, _P, _P]
        L.ref_save_training_checkpoint.restype = C.c_int
        L.ref_save_training_checkpoint.argtypes = cfg + [C.c_int] * 3 + [_I64, C.c_uint64, C.c_char_p, C.c_int]
        L.ref_sgd_step_f32.restype = C.c_int
        L.ref_sgd_step_f32.argtypes = [_P, _P, _P, _I64, C.c_double, C.c_double, C.c_double, C.c_int]
        L.ref_lr_at.restype = C.c_int
        L.ref_lr_at.argtypes = [C.c_int, C.c_double, C.c_int, _P, C.c_int, C.c_double, C.c_double, C.c_int,
                                C.POINTER(C.c_double)]
        L.ref_rng_normal.argtypes = [C.c_uint64, _I64, _P]
        L.ref_rng_u64.argtypes = [C.c_uint64, _I64, _P]
        L.ref_count_parameters.restype = C.c_int64
        L.ref_count_parameters.argtypes = cfg + [C.c_int]
        L.ref_preset_text.restype = C.c_int
        L.ref_preset_text.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.ref_config_roundtrip.restype = C.c_int
        L.ref_config_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.ref_parse_config.restype = C.c_int
        L.ref_parse_config.argtypes = [C.c_char_p, _P, C.c_int] + [_P] * 7
        L.ref_predict_peak_elements.restype = C.c_int
        L.ref_predict_peak_elements.argtypes = cfg + [C.c_int, _I64, C.c_int, C.c_int, C.c_int, _P]
        _ref[path] = L
    return _ref[path]


# ---------------------------------------------------------------------------
# flat layouts


@dataclass(frozen=True)
class BlockShape:
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

    def param_layer_size(self, l: int) -> int:
        c = self.c_in(l)
        return 2 * c + self.bk * c + 2 * self.bk + 9 * self.k * self.bk

    def param_offsets(self) -> list[int]:
        offs, o = [], 0
        for l in range(self.m):
            offs.append(o)
            o += self.param_layer_size(l)
        return offs

    @property
    def param_size(self) -> int:
        return sum(self.param_layer_size(l) for l in range(self.m))

    def stat_offsets(self) -> list[int]:
        offs, o = [], 0
        for l in range(self.m):
            offs.append(o)
            o += 2 * self.c_in(l) + 2 * self.bk
        return offs

    @property
    def stat_size(self) -> int:
        return sum(2 * self.c_in(l) + 2 * self.bk for l in range(self.m))

    def split_params(self, flat: np.ndarray) -> list[dict]:
        """Per-layer views {gamma_a, beta_a, w1, gamma_b, beta_b, w2}."""
        out = []
        for l, o in enumerate(self.param_offsets()):
            c, bk, k = self.c_in(l), self.bk, self.k
            d = {}
            d["gamma_a"] = flat[o:o + c]; o += c
            d["beta_a"] = flat[o:o + c]; o += c
            d["w1"] = flat[o:o + bk * c].reshape(bk, c); o += bk * c
            d["gamma_b"] = flat[o:o + bk]; o += bk
            d["beta_b"] = flat[o:o + bk]; o += bk
            d["w2"] = flat[o:o + 9 * k * bk].reshape(k, bk, 3, 3)
            out.append(d)
        return out

    def split_stats(self, flat: np.ndarray) -> list[dict]:
        out = []
        for l, o in enumerate(self.stat_offsets()):
            c, bk = self.c_in(l), self.bk
            out.append({"mean_a": flat[o:o + c], "var_a": flat[o + c:o + 2 * c],
                        "mean_b": flat[o + 2 * c:o + 2 * c + bk],
                        "var_b": flat[o + 2 * c + bk:o + 2 * c + 2 * bk]})
        return out

    def initial_running(self, dtype) -> np.ndarray:
        r = np.zeros(self.stat_size, dtype=dtype)
        for l, o in enumerate(self.stat_offsets()):
            c, bk = self.c_in(l), self.bk
            r[o + c:o + 2 * c] = 1
            r[o + 2 * c + bk:o + 2 * c + 2 * bk] = 1
        return r


def _suffix(dtype) -> str:
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


def rng_normal(seed: int, count: int, dtype=np.float64) -> np.ndarray:
    """Rng(seed).normal() x count (dp/rng.hpp:36-49), cast to dtype."""
    out = np.empty(count, dtype=np.float64)
    lib().dpo_fill_normal_f64(seed, _ptr(out), count)
    return out.astype(dtype)


def rng_u64(seed: int, count: int) -> np.ndarray:
    """Raw std::mt19937_64 draws of the restated engine."""
    out = np.empty(count, dtype=np.uint64)
    lib().dpo_rng_u64_fill(seed, _ptr(out), count)
    return out


def ref_rng_normal(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    ref_lib().ref_rng_normal(seed, count, _ptr(out))
    return out


def ref_rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    ref_lib().ref_rng_u64(seed, count, _ptr(out))
    return out


def block_forward(s: BlockShape, params, x_in, running=None, update_running=True):
    """Restated block forward.  Returns (feats, z, stats, running)."""
    dt = params.dtype
    feats = np.zeros((s.n, s.c_out, s.h, s.w), dtype=dt)
    feats[:, :s.c0] = x_in
    z = np.zeros((s.m, s.n, s.bk, s.h, s.w), dtype=dt)
    stats = np.zeros(s.stat_size, dtype=dt)
    run = s.initial_running(dt) if running is None else np.array(running, dtype=dt)
    rc = getattr(lib(), f"dpo_block_forward_{_suffix(dt)}")(
        s.n, s.h, s.w, s.c0, s.m, s.k, s.bk, _ptr(np.ascontiguousarray(params)),
        _ptr(feats), _ptr(z), _ptr(stats), _ptr(run), int(update_running))
    if rc != 0:
        raise RuntimeError(f"oracle block_forward status {rc}")
    return feats, z, stats, run


def block_backward(s: BlockShape, params, feats, z, stats, acc):
    """Restated block backward.  Returns (acc_out, grads)."""
    dt = params.dtype
    acc = np.array(acc, dtype=dt, order="C")
    grads = np.zeros(s.param_size, dtype=dt)
    rc = getattr(lib(), f"dpo_block_backward_{_suffix(dt)}")(
        s.n, s.h, s.w, s.c0, s.m, s.k, s.bk, _ptr(np.ascontiguousarray(params)),
        _ptr(np.ascontiguousarray(feats)), _ptr(np.ascontiguousarray(z)),
        _ptr(np.ascontiguousarray(stats)), _ptr(acc), _ptr(grads))
    if rc != 0:
        raise RuntimeError(f"oracle block_backward status {rc}")
    return acc, grads


def ref_block(s: BlockShape, params, x_in, acc=None, running=None, update_running=True):
    """The reference's own ops:: run through the block harness (oracle/_ref)."""
    dt = params.dtype
    L = ref_lib()
    feats = np.zeros((s.n, s.c_out, s.h, s.w), dtype=dt)
    z = np.zeros((s.m, s.n, s.bk, s.h, s.w), dtype=dt)
    stats = np.zeros(s.stat_size, dtype=dt)
    run = s.initial_running(dt) if running is None else np.array(running, dtype=dt)
    grads = np.zeros(s.param_size, dtype=dt)
    accv = None if acc is None else np.array(acc, dtype=dt, order="C")
    rc = getattr(L, f"ref_block_harness_{_suffix(dt)}")(
        s.n, s.h, s.w, s.c0, s.m, s.k, s.bk, _ptr(np.ascontiguousarray(params)),
        _ptr(np.ascontiguousarray(x_in, dtype=dt)), _ptr(run), int(update_running),
        _ptr(feats), _ptr(z), _ptr(stats), _ptr(accv), _ptr(grads))
    if rc != 0:
        raise RuntimeError(f"reference harness status {rc}: {L.ref_last_error().decode()}")
    return feats, z, stats, run, accv, grads


def random_block_params(s: BlockShape, seed: int, dtype=np.float32, perturb_bn=True) -> np.ndarray:
    """He-normal conv weights in reference draw order, BN gamma/beta either
    1/0 (reference init) or 1+0.5N / 0.5N (SURVEY §8(d) second parity case)."""
    flat = np.zeros(s.param_size, dtype=np.float64)
    draws = rng_normal(seed, 2 * s.param_size + 16)
    di = 0
    for l, o in enumerate(s.param_offsets()):
        c, bk, k = s.c_in(l), s.bk, s.k
        views = s.split_params(flat)[l]
        if perturb_bn:
            views["gamma_a"][:] = 1 + 0.5 * draws[di:di + c]; di += c
            views["beta_a"][:] = 0.5 * draws[di:di + c]; di += c
        else:
            views["gamma_a"][:] = 1
        views["w1"][:] = (draws[di:di + bk * c] * np.sqrt(2.0 / c)).reshape(bk, c); di += bk * c
        if perturb_bn:
            views["gamma_b"][:] = 1 + 0.5 * draws[di:di + bk]; di += bk
            views["beta_b"][:] = 0.5 * draws[di:di + bk]; di += bk
        else:
            views["gamma_b"][:] = 1
        views["w2"][:] = (draws[di:di + 9 * k * bk] * np.sqrt(2.0 / (9 * bk))).reshape(k, bk, 3, 3)
        di += 9 * k * bk
    return flat.astype(dtype)


# ---------------------------------------------------------------------------
# reference model-level helpers (need _ref)


def _cfg_args(blocks, k, bottleneck, compression, classes, c0):
    arr = (C.c_int * len(blocks))(*blocks)
    return [len(blocks), C.cast(arr, _P), k, int(bottleneck), float(compression), classes, c0], arr


def ref_count_parameters(blocks, k, bottleneck, compression, classes, c0, in_c=3) -> int:
    args, keep = _cfg_args(blocks, k, bottleneck, compression, classes, c0)
    return int(ref_lib().ref_count_parameters(*args, in_c))


def ref_predict_peak_elements(blocks, k, bottleneck, compression, classes, c0,
                              strategy, batch, in_c, in_h, in_w) -> list[int]:
    args, keep = _cfg_args(blocks, k, bottleneck, compression, classes, c0)
    out = np.zeros(6, dtype=np.int64)
    rc = ref_lib().ref_predict_peak_elements(*args, strategy, batch, in_c, in_h, in_w, _ptr(out))
    if rc != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return [int(v) for v in out]


def ref_block_params(blocks, k, bottleneck, compression, classes, c0, in_shape, seed, b) -> np.ndarray:
    """Block b's flat params exactly as GraphPlan<float>::build draws them."""
    args, keep = _cfg_args(blocks, k, bottleneck, compression, classes, c0)
    n, c, h, w = in_shape
    # size of block b
    cin = c0
    for bi, mb in enumerate(blocks):
        if bi == b:
            break
        cin = int(np.floor(compression * (cin + mb * k)))
    s = BlockShape(n, h, w, cin, blocks[b], k, 4 * k)
    out = np.zeros(s.param_size, dtype=np.float32)
    rc = ref_lib().ref_block_params_f32(*args, c, h, w, n, seed, b, _ptr(out))
    if rc != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return out


def ref_model_params(blocks, k, bottleneck, compression, classes, c0, in_shape, seed):
    """All parameters of GraphPlan<float>::build in registration order and the
    reference's synthetic NCHW input (Rng(seed+99).normal())."""
    args, keep = _cfg_args(blocks, k, bottleneck, compression, classes, c0)
    n, c, h, w = in_shape
    count = ref_lib().ref_count_parameters(*args, c)
    params = np.zeros(count, dtype=np.float32)
    x = np.zeros((n, c, h, w), dtype=np.float32)
    rc = ref_lib().ref_model_params_f32(*args, c, h, w, n, seed, _ptr(params), _ptr(x))
    if rc != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return params, x


def ref_model_grads(blocks, k, bottleneck, compression, classes, c0, in_shape, seed):
    """One GraphPlan<float>::step_trace: (loss, all parameter gradients in
    registration order).  Labels are i % classes (ref_driver make_labels)."""
    args, keep = _cfg_args(blocks, k, bottleneck, compression, classes, c0)
    n, c, h, w = in_shape
    count = ref_lib().ref_count_parameters(*args, c)
    grads = np.zeros(count, dtype=np.float32)
    loss = C.c_double()
    secs = C.c_double()
    rc = ref_lib().ref_model_step_f32(*args, c, h, w, n, seed, 1, C.byref(loss), C.byref(secs), _ptr(grads))
    if rc != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return loss.value, grads


def ref_model_step(blocks, k, bottleneck, compression, classes, c0, in_shape, seed,
                   steps=1, fast=False):
    """Times GraphPlan<float>::step_trace (the reference's public API).
    Returns (loss, best_seconds)."""
    args, keep = _cfg_args(blocks, k, bottleneck, compression, classes, c0)
    n, c, h, w = in_shape
    loss = C.c_double()
    secs = C.c_double()
    L = ref_lib(fast=fast)
    rc = L.ref_model_step_f32(*args, c, h, w, n, seed, steps, C.byref(loss), C.byref(secs), None)
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return loss.value, secs.value


def model_running_size(blocks, k, compression, c0, stem) -> int:
    """Running-statistics elements of the libdpb model layout (include/dpb.h)."""
    n, c = (2 * c0 if stem == 1 else 0), c0
    for b, m in enumerate(blocks):
        for l in range(m):
            n += 2 * (c + l * k) + 2 * 4 * k
        C = c + m * k
        n += 2 * C
        c = int(np.floor(compression * C))
    return n


def model_segments(blocks, k, compression, classes, c0, in_c=3, stem=0):
    """(name, elements) of every parameter tensor in libdpb's registration
    order (graph.hpp:405-600; the ImageNet stem's conv + BN first for stem=1)."""
    bk = 4 * k
    if stem == 1:
        segs = [("stem.conv.w", c0 * in_c * 49), ("stem.bn.gamma", c0), ("stem.bn.beta", c0)]
    else:
        segs = [("stem.conv.w", c0 * in_c * 9)]
    c = c0
    for b, m in enumerate(blocks):
        for l in range(m):
            ci = c + l * k
            segs += [(f"b{b}.l{l}.bn_a.gamma", ci), (f"b{b}.l{l}.bn_a.beta", ci), (f"b{b}.l{l}.conv_a.w", bk * ci),
                     (f"b{b}.l{l}.bn_b.gamma", bk), (f"b{b}.l{l}.bn_b.beta", bk), (f"b{b}.l{l}.conv_b.w", k * bk * 9)]
        C_ = c + m * k
        if b + 1 < len(blocks):
            cout = int(np.floor(compression * C_))
            segs += [(f"t{b}.bn.gamma", C_), (f"t{b}.bn.beta", C_), (f"t{b}.conv.w", cout * C_)]
            c = cout
        else:
            segs += [("head.bn.gamma", C_), ("head.bn.beta", C_), ("head.linear.w", classes * C_),
                     ("head.linear.b", classes)]
    return segs


def running_segments(blocks, k, compression, c0, stem=0):
    """(name, elements) of the running-statistics layout (include/dpb.h)."""
    bk = 4 * k
    segs = [("stem.bn.mean", c0), ("stem.bn.var", c0)] if stem == 1 else []
    c = c0
    for b, m in enumerate(blocks):
        for l in range(m):
            ci = c + l * k
            segs += [(f"b{b}.l{l}.bn_a.mean", ci), (f"b{b}.l{l}.bn_a.var", ci), (f"b{b}.l{l}.bn_b.mean", bk),
                     (f"b{b}.l{l}.bn_b.var", bk)]
        C_ = c + m * k
        nm = f"t{b}" if b + 1 < len(blocks) else "head"
        segs += [(f"{nm}.bn.mean", C_), (f"{nm}.bn.var", C_)]
        c = int(np.floor(compression * C_))
    return segs


def sketch(flat: np.ndarray, segs, nsample=256, nproj=4) -> dict:
    """Size-independent fingerprint of a flat tensor list, per segment: the
    2-norm, `nproj` projections onto fixed random +-1 vectors (their spread
    estimates ||a - b||, so sqrt(mean(dproj^2)) / ||b|| is an unbiased
    normwise-error estimate) and `nsample` elements at fixed indices."""
    norms, projs, idx, vals = [], [], [], []
    o = 0
    for i, (_, n) in enumerate(segs):
        seg = flat[o:o + n].astype(np.float64)
        norms.append(np.linalg.norm(seg))
        r = np.random.default_rng(7919 * i + 1)
        projs.append([float(np.dot(np.where(r.random(n) < 0.5, -1.0, 1.0), seg)) for _ in range(nproj)])
        take = np.arange(n) if n <= nsample else np.sort(r.choice(n, nsample, replace=False))
        idx.append(o + take)
        vals.append(flat[o + take])
        o += n
    assert o == flat.size
    return {"norm": np.array(norms), "proj": np.array(projs), "idx": np.concatenate(idx),
            "val": np.concatenate(vals)}


def sketch_errors(got: np.ndarray, ref_sketch: dict, segs):
    """Per-segment (normwise estimate from the projections, max elementwise
    rel_err over the sampled elements) of `got` against a stored sketch."""
    g = sketch(got, segs, nproj=ref_sketch["proj"].shape[1])
    dproj = g["proj"] - ref_sketch["proj"]
    est = np.sqrt(np.mean(dproj ** 2, axis=1)) / np.maximum(ref_sketch["norm"], 1e-30)
    a = got[ref_sketch["idx"]].astype(np.float64)
    b = ref_sketch["val"].astype(np.float64)
    rel = np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return est, rel


def ref_single_block_trace(m, k, c0, n, h, w, seed=5, strategy=2):
    """The reference's OpTrace of one GraphPlan<double> step of the single-block
    network blocks={m} (4 classes): (counts [nodes, 3] = forward, backward,
    recompute; flops [3, 7] = forward / backward / recompute per OpKind)."""
    L = ref_lib()
    f = L.ref_single_block_trace
    f.restype = C.c_int
    f.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_int, _P, C.c_int, _P, C.POINTER(C.c_int)]
    counts = np.zeros(3 * 4096, dtype=np.int32)
    flops = np.zeros(21, dtype=np.float64)
    nn = C.c_int()
    rc = f(m, k, c0, n, h, w, seed, strategy, _ptr(counts), 4096, _ptr(flops), C.byref(nn))
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return counts[:3 * nn.value].reshape(-1, 3), flops.reshape(3, 7)


def block_trace_flops(s: "BlockShape"):
    """Per-kind FLOPs of one dense block under the reference's conventions
    (ops.hpp:565-595): forward / backward / one rematerialisation per layer
    (concat, bn_a, relu_a over c channels; bn_b, relu_b over bk), as
    GraphPlan::forward_layer / backward_layer / rematerialize count them."""
    M = s.n * s.h * s.w
    fwd = np.zeros(7)
    bwd = np.zeros(7)
    rem = np.zeros(7)
    for l in range(s.m):
        c = s.c_in(l)
        f1, f3 = 2.0 * M * s.bk * c, 2.0 * M * s.k * 9 * s.bk
        fwd[0] += M * c
        fwd[1] += 8.0 * M * (c + s.bk)
        fwd[2] += M * (c + s.bk)
        fwd[3] += f1 + f3
        bwd[0] += M * c
        bwd[1] += 12.0 * M * (c + s.bk)
        bwd[2] += M * (c + s.bk)
        bwd[3] += 2.0 * (f1 + f3)
        rem[0] += M * c
        rem[1] += 8.0 * M * (c + s.bk)
        rem[2] += M * (c + s.bk)
    fwd[0] += M * s.c_out  # block-output concat
    return fwd, bwd, rem


def ref_model_train_step(blocks, k, compression, classes, c0, in_shape, seed, stem=0, params=None, x=None,
                         dtype=np.float32):
    """One reference training step through GraphPlan<T>'s public forward /
    compute_loss / backward (ref_model_train_step_f32/_f64 in ref_driver.cpp),
    composed with the ImageNet stem for stem=1.  Returns (loss, grads,
    running) in libdpb's flat layouts, in `dtype`.  params (float32) None =
    GraphPlan<float>::build's init (stem 0, float32 only); x None = the float
    input Rng(seed + 99).normal() (exact in float64 too)."""
    L = ref_lib()
    n, c, h, w = in_shape
    count = ref_count_parameters(blocks, k, True, compression, classes, c0, c)
    if stem == 1:
        count += c0 * c * 49 - c0 * c * 9 + 2 * c0
    if params is not None:
        assert params.size == count and params.dtype == np.float32, (params.size, count, params.dtype)
    if dtype == np.float64 and params is None:
        raise ValueError("the float64 reference step needs explicit (float32) parameters")
    grads = np.zeros(count, dtype=dtype)
    running = np.zeros(model_running_size(blocks, k, compression, c0, stem), dtype=dtype)
    loss = C.c_double()
    arr = (C.c_int * len(blocks))(*blocks)
    f = getattr(L, f"ref_model_train_step_{_suffix(dtype)}")
    f.restype = C.c_int
    f.argtypes = [C.c_int, _P, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _I64,
                  C.c_uint64, _P, _P, C.POINTER(C.c_double), _P, _P]
    xx = None if x is None else np.ascontiguousarray(x, dtype=np.float32)
    pp = None if params is None else np.ascontiguousarray(params)
    rc = f(len(blocks), C.cast(arr, _P), k, compression, classes, c0, stem, c, h, w, n, seed, _ptr(pp), _ptr(xx),
           C.byref(loss), _ptr(grads), _ptr(running))
    if rc != 0:
        raise RuntimeError(f"reference train step status {rc}: {L.ref_last_error().decode()}")
    return loss.value, grads, running


# ---- optimizer -------------------------------------------------------
def sgd_step(p, g, v, lr, momentum, weight_decay, nesterov):
    """train.hpp:43-70 restated in float32 numpy (every op rounded, no FMA):
    d = g + wd*p; v = mu*v + d; p -= lr*(nesterov ? d + mu*v : v).  In place."""
    f = np.float32
    mu, wd, eta = f(momentum), f(weight_decay), f(lr)
    d = g + wd * p
    v[:] = mu * v + d
    p -= eta * ((d + mu * v) if nesterov else v)


def ref_sgd_step(p, g, v, lr, momentum, weight_decay, nesterov):
    """The reference's own sgd_step (oracle/_ref), in place."""
    rc = ref_lib().ref_sgd_step_f32(_ptr(p), _ptr(g), _ptr(v), p.size, lr, momentum, weight_decay, int(nesterov))
    if rc != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())


def lr_at(kind, base_lr, total_epochs, epoch, milestones=(), factor=0.1, floor=0.0):
    """schedule.hpp:46-62 restated."""
    if not 0 <= epoch < total_epochs:
        raise ValueError("epoch out of range")
    if kind == "cosine":
        return floor + (base_lr - floor) / 2.0 * (np.cos(np.pi * epoch / total_epochs) + 1.0)
    lr = base_lr
    for m in milestones:
        if epoch >= m:
            lr *= factor
    return lr


def ref_lr_at(kind, base_lr, total_epochs, epoch, milestones=(), factor=0.1, floor=0.0):
    arr = (C.c_int * max(1, len(milestones)))(*milestones)
    out = C.c_double()
    rc = ref_lib().ref_lr_at({"step": 0, "cosine": 1}[kind], base_lr, total_epochs, C.cast(arr, C.c_void_p),
                             len(milestones), factor, floor, epoch, C.byref(out))
    if rc != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return out.value


def ref_save_training_checkpoint(blocks, k, compression, classes, c0, in_shape, seed, path, epoch):
    """The reference writes a DPLN training checkpoint (velocities 0.5 * params)."""
    args, keep = _cfg_args(blocks, k, 1, compression, classes, c0)
    n, c, h, w = in_shape
    rc = ref_lib().ref_save_training_checkpoint(*args, c, h, w, n, seed, path.encode(), epoch)
    if rc != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())


def ref_preset_text(name: str):
    """config_to_text(preset_config(name)) from the reference, or (status, message)."""
    buf = C.create_string_buffer(4096)
    rc = ref_lib().ref_preset_text(name.encode(), buf, len(buf))
    if rc:
        return {"status": rc, "message": ref_lib().ref_last_error().decode()}
    return {"text": buf.value.decode()}


def ref_parse_config(text: str):
    """The reference's config_from_key_values(parse_key_values(text)) as a dict,
    or its error {status, message} (status = errors.hpp class index)."""
    blocks = np.zeros(64, dtype=np.int32)
    ints = [C.c_int() for _ in range(6)]
    comp = C.c_double()
    nb, k, bott, c0, post, classes = ints
    rc = ref_lib().ref_parse_config(text.encode(), C.c_void_p(blocks.ctypes.data), 64, C.byref(nb), C.byref(k),
                                    C.byref(bott), C.byref(comp), C.byref(c0), C.byref(post), C.byref(classes))
    if rc:
        return {"status": rc, "message": ref_lib().ref_last_error().decode()}
    return {"blocks": [int(b) for b in blocks[:nb.value]], "growth_rate": k.value, "bottleneck": bool(bott.value),
            "compression": comp.value, "initial_channels": c0.value,
            "activation": "post" if post.value else "pre", "num_classes": classes.value}


def ref_config_roundtrip(text: str):
    """config_to_text of the reference's parse of `text`, or its error."""
    buf = C.create_string_buffer(4096)
    rc = ref_lib().ref_config_roundtrip(text.encode(), buf, len(buf))
    if rc:
        return {"status": rc, "message": ref_lib().ref_last_error().decode()}
    return {"text": buf.value.decode()}
