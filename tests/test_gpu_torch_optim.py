"""The torch.optim front end: autograd gradients on a real model feed the fused step.

A small MLP trained with WagmaSGD on one GPU (P = 1 rank, S = 1) for a few
iterations incl. global syncs must land bit-exactly where the oracle's Alg. 2
replay lands with the same (recorded) gradients; parameters stay views of the
replica buffer the kernel updates.
"""

import numpy as np
import pytest
import torch

from oracle import wagma_oracle as wo
from paper_2005_00124_b200.context import DeviceContext
from paper_2005_00124_b200.optim import EtaSchedule, OptimizerConfig
from paper_2005_00124_b200.torch_optim import WagmaSGD, flat_numel

pytestmark = pytest.mark.gpu


def test_wagma_sgd_matches_oracle(cuda):
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(16, 33), torch.nn.Tanh(), torch.nn.Linear(33, 5)).cuda()
    n = flat_numel(model.parameters())
    T, tau = 7, 3
    ctx = DeviceContext(1, 1, n, tau=tau, timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=1, tau=tau, eta=EtaSchedule(value=0.05), update_rule="momentum", momentum=0.9)
    opt = WagmaSGD(model.parameters(), ctx, cfg)
    w0 = opt.flat.detach().cpu().numpy().copy()
    grads = []
    x = torch.randn(64, 16, device="cuda")
    y = torch.randn(64, 5, device="cuda")
    for _ in range(T):
        opt.zero_grad()
        loss = torch.nn.functional.mse_loss(model(x), y)
        loss.backward()
        grads.append(opt.flat_grad.detach().cpu().numpy().copy())
        opt.step()
    torch.cuda.synchronize()
    ctx.check()
    # parameters are still views of the replica the kernel wrote
    first = next(model.parameters())
    assert first.data_ptr() == opt.flat.data_ptr()
    stamps = np.array([[t] for t in range(T)], dtype=np.int64)
    want = wo.replay_training(P=1, S=1, tau=tau, T=T, w0=w0, grads=np.stack(grads)[:, None, :],
                              etas=np.full((T, 1), 0.05), stamps=stamps, update_rule="momentum",
                              momentum=0.9, dtype=np.float32)
    assert np.array_equal(opt.flat.cpu().numpy(), want[0])
    ctx.close()
