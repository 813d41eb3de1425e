"""The native data-parallel path on one GPU: libdpb's NCCL
communicator attached to a ModelPlan.  With one rank the per-bucket ncclAvg
allreduces are identities, so the step must reproduce the communicator-free
step bit for bit — through the communication stream, its events and the
CUDA-graph capture (the multi-rank exchange itself runs under torchrun in
bench.py; the bucket schedule is checked on CPU in tests/test_dp.py)."""
import numpy as np
import pytest
import torch

from paper_1707_06990_b200.dp import DpComm, model_buckets
from paper_1707_06990_b200.model import DenseNetConfig, ModelPlan, init_params, model_sizes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("stem", ["3x3", "imagenet"])
def test_single_rank_comm_step_is_identity(stem):
    shape = (3, 16, 16) if stem == "3x3" else (3, 33, 35)
    cfg = DenseNetConfig((2, 3, 2), 8, True, 0.5, 10, 16, shape, stem=stem)
    n = 4
    x = torch.randn(n, *shape, generator=torch.Generator().manual_seed(3)).cuda()
    labels = (torch.arange(n, dtype=torch.int32) % 10).cuda()
    params = torch.from_numpy(init_params(cfg, 5)).cuda()
    out = []
    for use_comm in (False, True):
        st = torch.cuda.Stream()
        plan = ModelPlan(cfg, n, dtype="bf16", stream=st)
        comm = DpComm(0, 1, torch.cuda.current_device()) if use_comm else None
        plan.set_comm(comm)
        run = plan.initial_running()
        grads = torch.empty(plan.param_elems, device="cuda")
        loss = torch.zeros(1, device="cuda")
        for _ in range(3):  # capture, then replay
            plan.step(x, labels, params, run, grads, loss)
        plan.sync()
        torch.cuda.synchronize()
        if comm is not None:
            comm.check()
        out.append((grads.cpu().numpy(), loss.item()))
        plan.close()
        if comm is not None:
            comm.close()
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]


def test_buckets_tile_the_parameters():
    cfg = DenseNetConfig((6, 12, 64, 48), 32, True, 0.5, 1000, 64, (3, 224, 224), stem="imagenet")
    b = model_buckets(cfg)
    assert len(b) == 4 and b[-1][0] == 0 and b[0][1] == model_sizes(cfg)[0]
    assert all(b[i][0] == b[i + 1][1] for i in range(len(b) - 1))
