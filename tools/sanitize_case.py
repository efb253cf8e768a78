"""Small single-GPU run for compute-sanitizer (racecheck / synccheck / memcheck).

P=4 ranks, S=2 and S=4 plans, tau=3 (one global sync), n = 3 tiles + a
ragged end, emulated straggler (mixed versions, stale leaves), on the TMA
kernel (default) or the cp.async kernel (WG_LOC=0). Exits 0 and prints
"sanitize case ok" when the device results match the oracle.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import wagma_oracle as wo  # noqa: E402  (checker only)
from paper_2005_00124_b200.context import DeviceContext  # noqa: E402
from paper_2005_00124_b200.driver import TickSchedule, contribution_log  # noqa: E402
from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig  # noqa: E402
from paper_2005_00124_b200.straggler import StragglerPolicy  # noqa: E402


def run(P, S, tau, T, n):
    g = torch.Generator().manual_seed(5)
    grads = torch.randn(T, P, n, generator=g) * 0.01
    w0 = torch.randn(n, generator=g) * 0.02
    ctx = DeviceContext(P, S, n, tau=tau, version_ring=T, timeout_s=30.0)
    cfg = OptimizerConfig(T=T, S=S, tau=tau, eta=EtaSchedule(value=0.05), update_rule="momentum")
    opt = GroupAveragingOptimizer(ctx, cfg, w0.cuda())
    dg = grads.cuda()
    pol = StragglerPolicy(1, 1.0, selection_seed=2)
    TickSchedule(P, T, tau, lambda t: pol.victims(t, P)).run(opt, lambda r, t: dg[t, r])
    torch.cuda.synchronize()
    ctx.check()
    want = wo.replay_training(P=P, S=S, tau=tau, T=T, w0=w0.numpy(), grads=grads.numpy(),
                              etas=np.full((T, P), 0.05), stamps=contribution_log(ctx, T, tau),
                              update_rule="momentum", momentum=0.9, dtype=np.float32)
    got = np.stack([opt.W[r].cpu().numpy() for r in range(P)])
    assert np.array_equal(got, want)
    ctx.close()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    run(4, 2, 3, 5, 3 * 2048 + 5)
    run(4, 4, 3, 4, 2048)
    print("sanitize case ok")
