"""B200-native memory-efficient DenseNet dense block (arXiv 1707.06990).

Drop-in for the dense-block hot path of the reference ``denseplan`` library:
``BlockPlan`` (forward / backward over a per-block HBM arena), ``ops`` (the
per-op surface of ops.hpp), and the host-side model arithmetic.  All compute
runs in ``_build/libdpb.so`` (hand-written CUDA for sm_100a).
"""
from . import errors
from .block import BlockPlan, BlockShape, block_memory, plan_arena
from .naive import NaiveBlock
from .model import CONFIGS, DenseNetConfig, ModelPlan, count_parameters, predict_peak_elements, rng_normal

__all__ = ["errors", "BlockPlan", "BlockShape", "block_memory", "plan_arena", "CONFIGS",
           "DenseNetConfig", "ModelPlan", "NaiveBlock", "count_parameters", "predict_peak_elements", "rng_normal"]
