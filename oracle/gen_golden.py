"""TEST INFRASTRUCTURE — regenerates tests/golden/*.npz from the reference.

Run in the build container (needs /root/reference, i.e. oracle/_ref):

    python -m oracle.gen_golden

Every fixture is produced by the UNMODIFIED reference headers compiled into
oracle/_ref/libdenseplan_ref.so: the block-level harness over the public
``ops::`` functions (itself checked bitwise against GraphPlan::step_trace by
``ref_check_block_harness``), ``GraphPlan::build`` parameter draws,
``count_parameters`` and ``predict_peak_elements``.  The fixtures are small
(<1 MB total) and committed; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import json
import sys
import os

import numpy as np

from oracle import oracle as O

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

# name -> (BlockShape, params source, dtype)
CASES = {
    # perturbed BN gamma/beta (SURVEY §8(d) second parity case)
    "small_perturbed_f32": (O.BlockShape(2, 5, 6, 8, 3, 4, 16), "perturbed", np.float32),
    "small_perturbed_f64": (O.BlockShape(2, 5, 6, 8, 3, 4, 16), "perturbed", np.float64),
    # ragged: odd spatial dims, odd channel counts
    "ragged_f32": (O.BlockShape(3, 7, 3, 5, 2, 3, 12), "perturbed", np.float32),
    # minimum non-degenerate batch: n*h*w == 2 (ops.hpp:180-183)
    "minimal_f32": (O.BlockShape(1, 1, 2, 4, 1, 2, 8), "perturbed", np.float32),
    # parameters exactly as GraphPlan<float>::build draws them for a
    # single-block model blocks={4}, k=4, c0=8 (He-normal; gamma=1, beta=0)
    "graphplan_init_f32": (O.BlockShape(2, 6, 6, 8, 4, 4, 16), "graphplan", np.float32),
    # the cfg1 channel geometry (c0=24, k=12, bk=48) at a reduced batch/field
    "cfg1_geometry_f32": (O.BlockShape(2, 8, 8, 24, 3, 12, 48), "perturbed", np.float32),
}


def make_case(name, s, src, dt):
    seed = 7
    if src == "graphplan":
        params = O.ref_block_params([s.m], s.k, True, 1.0, 4, s.c0, (s.n, 3, s.h, s.w), seed, 0)
    else:
        params = O.random_block_params(s, seed, dt, perturb_bn=True)
    params = params.astype(dt)
    x_in = O.rng_normal(seed + 99, s.n * s.c0 * s.h * s.w, dt).reshape(s.n, s.c0, s.h, s.w)
    acc_in = O.rng_normal(seed + 100, s.n * s.c_out * s.h * s.w, dt).reshape(s.n, s.c_out, s.h, s.w)
    # running stats start from a non-trivial state so the momentum rule is exercised
    running_in = s.initial_running(dt)
    running_in += (0.25 * O.rng_normal(seed + 101, running_in.size)).astype(dt)
    running_in = np.abs(running_in).astype(dt)
    feats, z, stats, running, acc_out, grads = O.ref_block(s, params, x_in, acc_in, running_in, True)
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        shape=np.array([s.n, s.h, s.w, s.c0, s.m, s.k, s.bk], dtype=np.int64),
        params=params, x_in=x_in, acc_in=acc_in, running_in=running_in,
        feats=feats, z=z, stats=stats, running=running, acc_out=acc_out, grads=grads)


def kats():
    """Known-answer values pinned by the reference's own tests, recomputed
    by the reference code here (t/densenet_test.cpp:214-231,
    t/alloctrace_test.cpp:85-124)."""
    d = {}
    d["count_parameters"] = {
        "bc100_k12": O.ref_count_parameters([16, 16, 16], 12, True, 0.5, 10, 24),
        "d121_k32": O.ref_count_parameters([6, 12, 24, 16], 32, True, 0.5, 1000, 64),
        "d264_k32": O.ref_count_parameters([6, 12, 64, 48], 32, True, 0.5, 1000, 64),
        "d264_k48": O.ref_count_parameters([6, 12, 64, 48], 48, True, 0.5, 1000, 96),
        "bc160_k12": O.ref_count_parameters([26, 26, 26], 12, True, 0.5, 10, 24),
        "paper264_k48_preset": O.ref_count_parameters([6, 32, 64, 48], 48, True, 0.5, 1000, 96),
        "paper264_k32_preset": O.ref_count_parameters([6, 32, 64, 48], 32, True, 0.5, 1000, 64),
    }
    peaks = {}
    cfgs = {
        "tiny_block_k2": ([3], 2, False, 1.0, 2, 2, 1, 1, 4, 4),  # alloctrace_test KAT
        "cfg1": ([12], 12, True, 1.0, 10, 24, 16, 3, 32, 32),
        "bc100_b64": ([16, 16, 16], 12, True, 0.5, 10, 24, 64, 3, 32, 32),
        "d121_b64_56": ([6, 12, 24, 16], 32, True, 0.5, 1000, 64, 64, 3, 56, 56),
        "d264k32_b64_56": ([6, 12, 64, 48], 32, True, 0.5, 1000, 64, 64, 3, 56, 56),
        "d264k48_b64_56": ([6, 12, 64, 48], 48, True, 0.5, 1000, 96, 64, 3, 56, 56),
    }
    for name, (blocks, k, bott, comp, classes, c0, n, c, h, w) in cfgs.items():
        peaks[name] = {strat: O.ref_predict_peak_elements(blocks, k, bott, comp, classes, c0,
                                                          si, n, c, h, w)
                       for si, strat in enumerate(["naive", "shared_grad", "shared_all"])}
    d["predict_peak_elements"] = peaks
    # denseplan::Rng (the reference's own engine + Box-Muller)
    d["rng_u64_seed7_first4"] = [int(v) for v in O.ref_rng_u64(7, 4)]
    d["rng_normal_seed106_first8"] = [float(v) for v in O.ref_rng_normal(106, 8)]
    # GraphPlan::build's parameters at DenseNet-264 scale (tests/test_model_host.py)
    import hashlib
    d["params_sha256_seed7"] = {}
    for name, (k, c0) in {"d264k32@56": (32, 64), "d264k48@56": (48, 96)}.items():
        p, _ = O.ref_model_params([6, 12, 64, 48], k, 1, 0.5, 1000, c0, (1, 3, 56, 56), 7)
        d["params_sha256_seed7"][name] = hashlib.sha256(p.tobytes()).hexdigest()
    # the reference's OpTrace of a single-block network (tests/test_trace*.py)
    counts, flops = O.ref_single_block_trace(3, 4, 8, 2, 5, 6, strategy=2)
    d["block_trace_m3k4c8_n2h5w6"] = {"counts": counts.tolist(), "flops": flops.tolist()}
    return d


# Whole-network training steps: the reference's own
# GraphPlan<float>::build parameters, synthetic input Rng(seed+99), labels
# i % classes, and one step_trace's loss and gradients (registration order).
MODEL_CASES = {
    # blocks, k, compression, classes, c0, (n, c, h, w), seed
    "model_small": ((2, 2, 2), 4, 0.5, 10, 8, (4, 3, 8, 8), 7),
    "model_bc": ((3, 3, 3), 12, 0.5, 10, 24, (8, 3, 16, 16), 11),
    # k = 32 (DenseNet-121 / 264-k32 growth, bk = 128): per-tap 3x3 kernels, bk > 64 1x1 variants
    "model_k32": ((2, 2), 32, 0.5, 10, 64, (4, 3, 8, 8), 13),
    # odd spatial size: 9x9 -> the transition pools (9-2)/2+1 = 4, so the pooling
    # windows do not tile the input (the partial-window backward path)
    "model_odd": ((2, 2), 8, 0.5, 10, 16, (4, 3, 9, 9), 17),
}


def make_model_case(name, blocks, k, comp, classes, c0, in_shape, seed):
    params, x = O.ref_model_params(blocks, k, 1, comp, classes, c0, in_shape, seed)
    loss, grads = O.ref_model_grads(blocks, k, 1, comp, classes, c0, in_shape, seed)
    labels = (np.arange(in_shape[0]) % classes).astype(np.int32)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), blocks=np.array(blocks), k=k, compression=comp,
                        classes=classes, c0=c0, in_shape=np.array(in_shape), seed=seed, params=params,
                        x=x, labels=labels, loss=np.float64(loss), grads=grads)


# Whole-network training steps with BN running statistics (F10), through the
# reference's public forward / compute_loss / backward (ref_model_train_step).
# Small cases store everything; the BASELINE-scale ones store per-tensor
# sketches (norm, random projections, sampled elements: oracle.sketch).
# Parameters are GraphPlan::build's for `seed` (libdpb replays them bit for
# bit: tests/test_model_host.py); the ImageNet-stem cases use libdpb's init
# for the stem-extended layout (dpb_model_init_params).  Input Rng(seed+99).
TRAIN_CASES = {
    # name: blocks, k, compression, classes, c0, (n, c, h, w), seed, stem, full
    "train_small": ((2, 2, 2), 4, 0.5, 10, 8, (4, 3, 8, 8), 7, 0, True),
    "train_imagenet_small": ((2, 2), 4, 0.5, 10, 8, (2, 3, 17, 19), 5, 1, True),
    "train_imagenet_k32": ((2, 2), 32, 0.5, 10, 64, (2, 3, 32, 32), 9, 1, True),
    # BASELINE configs[1]: DenseNet-BC-100 at its bench shape
    "train_bc100_b64": ((16, 16, 16), 12, 0.5, 10, 24, (64, 3, 32, 32), 7, 0, True),
    # BASELINE configs[3] / [4] in the reference's geometry (3x56x56)
    "train_d264k32_56": ((6, 12, 64, 48), 32, 0.5, 1000, 64, (2, 3, 56, 56), 7, 0, False),
    "train_d264k48_56": ((6, 12, 64, 48), 48, 0.5, 1000, 96, (2, 3, 56, 56), 7, 0, False),
    # the bench headline network: DenseNet-264-k32 with the ImageNet stem at 224x224
    "train_d264k32_224": ((6, 12, 64, 48), 32, 0.5, 1000, 64, (2, 3, 224, 224), 7, 1, False),
    # BASELINE configs[2]: DenseNet-121 with the ImageNet stem at 224x224
    "train_d121_224": ((6, 12, 24, 16), 32, 0.5, 1000, 64, (2, 3, 224, 224), 11, 1, False),
}


def make_train_case(name, blocks, k, comp, classes, c0, in_shape, seed, stem, full):
    """The reference step in float32 (GraphPlan<float>, the reference as
    shipped) and float64 (GraphPlan<double> on the same float parameters and
    input: the exact-arithmetic yardstick), plus the float32 reference's own
    per-tensor deviation from float64 (its precision noise: ReLU-mask flips
    near zero, long sequential sums; tests/test_train_gpu.py)."""
    n, c, h, w = in_shape
    if stem == 1:
        sys.path.insert(0, os.path.dirname(OUT.rstrip("/").rsplit("/", 1)[0]))
        from paper_1707_06990_b200.model import DenseNetConfig, init_params
        params = init_params(DenseNetConfig(tuple(blocks), k, True, comp, classes, c0, (c, h, w), stem="imagenet"),
                             seed)
    else:
        params, _ = O.ref_model_params(blocks, k, 1, comp, classes, c0, in_shape, seed)
    loss, grads, running = O.ref_model_train_step(blocks, k, comp, classes, c0, in_shape, seed, stem, params)
    loss64, grads64, running64 = O.ref_model_train_step(blocks, k, comp, classes, c0, in_shape, seed, stem, params,
                                                        dtype=np.float64)
    gsegs = O.model_segments(blocks, k, comp, classes, c0, c, stem)
    rsegs = O.running_segments(blocks, k, comp, c0, stem)

    def noise(a32, a64, segs):  # per tensor: normwise and max elementwise rel_err of float32 vs float64
        nw, el, o = [], [], 0
        for _, m in segs:
            x, y = a32[o:o + m].astype(np.float64), a64[o:o + m]
            nw.append(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))
            el.append(float(np.max(np.abs(x - y) / np.maximum(1.0, np.maximum(np.abs(x), np.abs(y))))))
            o += m
        return np.array(nw), np.array(el)

    gn, ge = noise(grads, grads64, gsegs)
    rn, re_ = noise(running, running64, rsegs)
    meta = dict(blocks=np.array(blocks), k=k, compression=comp, classes=classes, c0=c0, in_shape=np.array(in_shape),
                seed=seed, stem=stem, loss=np.float64(loss), loss64=np.float64(loss64),
                grads_noise=gn, grads_noise_el=ge, running_noise=rn, running_noise_el=re_,
                grads_noise_all=np.linalg.norm(grads - grads64) / np.linalg.norm(grads64))
    if full:
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), grads64=grads64, running64=running64, **meta)
        return
    sk = {}
    for tag, arr, segs in (("grads", grads, gsegs), ("grads64", grads64, gsegs), ("running", running, rsegs),
                           ("running64", running64, rsegs)):
        sk.update({f"{tag}_{key}": v for key, v in O.sketch(arr, segs).items()})
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **meta, **sk,
                        grads64_norm_all=np.float64(np.linalg.norm(grads64)))


# Config text KATs (densenet.hpp:86-115, 276-377): every preset through
# config_to_text, and texts through config_from_key_values(parse_key_values),
# including the reference's error class and message for the malformed ones.
CONFIG_PRESETS = ["desk", "tiny", "paper-264-k48", "paper-264-k32", "paper-232-k48", "bc-160-k12", "nope"]
CONFIG_TEXTS = [
    "",
    "blocks=16,16,16\ngrowth_rate=12\nbottleneck=1\ncompression=0.5\ninitial_channels=24\n"
    "activation=pre\nnum_classes=10\n",
    "  # comment line\n\nblocks=6,12 # trailing comment\n  growth_rate=32  \n\tbottleneck=1\r\n",
    "blocks = 1",
    "blocks=1,,2",
    "blocks=1,2,",
    "blocks=,1",
    "blocks=1\ngarbage",
    "blocks=1\ngrowth_rate=abc",
    "blocks=1\ngrowth_rate=12abc",
    "blocks=1\ncompression=1.5",
    "blocks=1\ncompression=0.25e0",
    "blocks=1\ncompression=.75",
    "blocks=1\ncompression=0x1p-2",
    "blocks=1\ncompression=nan",
    "blocks=1\ncompression=inf",
    "blocks=1\ncompression=1e999",
    "blocks=1\ncompression=x",
    "blocks=1\nactivation=mid",
    "blocks=1\nactivation=post",
    "blocks=0",
    "blocks=2\nbottleneck=7",
    "blocks=3\nblocks=4",
    "blocks=+3",
    "blocks= 3",
    "blocks=3 ,4",
    "growth_rate=-1\nblocks=1",
    "initial_channels=0\nblocks=1",
    "num_classes=0\nblocks=1",
    "a=b=c\nblocks=1",
    "=5\nblocks=1",
    "blocks=99999999999",
    "growth_rate=99999999999\nblocks=1",
    "blocks=2,2\ngrowth_rate=8\ncompression=0.333333333\ninitial_channels=-5",
    "blocks=1\nnum_classes=1000\ncompression=1",
    "blocks=2,2\ngrowth_rate=8\ncompression=0.333333333\ninitial_channels=5",
    "blocks=2\ncompression=0.1234567",
    "blocks=2\ncompression=1e-7",
]


def config_kats():
    presets = {name: O.ref_preset_text(name) for name in CONFIG_PRESETS}
    texts = [{"text": t, "result": O.ref_parse_config(t), "roundtrip": O.ref_config_roundtrip(t)}
             for t in CONFIG_TEXTS]
    return {"presets": presets, "texts": texts}


def main():
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "config_kats.json"), "w") as f:
        json.dump(config_kats(), f, indent=1, sort_keys=True)
    if "--config-only" in sys.argv:
        return
    if "--train" in sys.argv:  # one training-step case: python -m oracle.gen_golden --train NAME
        name = sys.argv[sys.argv.index("--train") + 1]
        make_train_case(name, *TRAIN_CASES[name])
        return
    if "--model" in sys.argv:  # one model case only: python -m oracle.gen_golden --model NAME
        name = sys.argv[sys.argv.index("--model") + 1]
        make_model_case(name, *MODEL_CASES[name])
        return
    for name, (s, src, dt) in CASES.items():
        make_case(name, s, src, dt)
    for name, args in MODEL_CASES.items():
        make_model_case(name, *args)
    for name, args in TRAIN_CASES.items():
        make_train_case(name, *args)
    with open(os.path.join(OUT, "kats.json"), "w") as f:
        json.dump(kats(), f, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
