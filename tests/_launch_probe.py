"""Helper of tests/test_launch_modes_gpu.py: one whole-network training step
(model_bc golden inputs, bf16) through ModelPlan on a created stream, written
to argv[1] as .npz.  Run in a fresh process per launch mode, since the library
reads DPB_NO_PDL / DPB_NO_FORK once per process."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_06990_b200.model import DenseNetConfig, ModelPlan  # noqa: E402

g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "model_bc.npz"))
n, cin, h, w = (int(v) for v in g["in_shape"])
cfg = DenseNetConfig(tuple(int(b) for b in g["blocks"]), int(g["k"]), True, float(g["compression"]),
                     int(g["classes"]), int(g["c0"]), (cin, h, w))
stream = torch.cuda.Stream()
plan = ModelPlan(cfg, n, dtype="bf16", stream=stream)
params = torch.from_numpy(g["params"]).cuda()
x = torch.from_numpy(g["x"]).cuda()
labels = torch.from_numpy(g["labels"]).cuda()
running = plan.initial_running()
grads = torch.empty(plan.param_elems, device="cuda")
loss = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
for _ in range(3):  # the first call captures the step's graph, the others replay it
    plan.step(x, labels, params, running, grads, loss)
    plan.sync()
torch.cuda.synchronize()
np.savez(sys.argv[1], grads=grads.cpu().numpy(), loss=loss.cpu().numpy(), running=running.cpu().numpy())
plan.close()
