"""One rank of a multi-GPU WAGMA run (launched by torchrun from test_gpu_multi.py).

Each process owns one GPU and P/G WAGMA ranks; send rings are mapped across
processes with CUDA IPC, so the fused kernel pulls peer replicas over
NVLink. Victim GPUs of `StragglerPolicy.victims` get a device-side delay
before their step, so the live activation protocol really sees stragglers.
Every process writes its replicas and gradients; rank 0 also writes the
device contribution log. The parent test replays them through the oracle.
"""

import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2005_00124_b200.context import DeviceContext  # noqa: E402
from paper_2005_00124_b200.driver import contribution_log, synthetic_grad  # noqa: E402
from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig  # noqa: E402
from paper_2005_00124_b200.straggler import StragglerPolicy  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--S", type=int, default=2)
    ap.add_argument("--T", type=int, default=20)
    ap.add_argument("--tau", type=int, default=5)
    ap.add_argument("--nelem", type=int, default=10007)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--victims", type=int, default=1)
    ap.add_argument("--delay-us", type=float, default=2000.0)
    ap.add_argument("--grace-us", type=float, default=50.0)
    ap.add_argument("--momentum", type=int, default=1)
    ap.add_argument("--alpha", type=int, default=1)
    ap.add_argument("--pipelined", type=int, default=0,
                    help="launch steps back to back (no host synchronisation per step, as bench.py does)")
    ap.add_argument("--save-grads", type=int, default=1,
                    help="0: the parent regenerates the gradients (driver.synthetic_grad) instead of loading them")
    a = ap.parse_args()

    rank = int(os.environ["RANK"])
    G = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    dt = torch.float32 if a.dtype == "f32" else torch.float64
    ctx = DeviceContext(a.P, a.S, a.nelem, dtype=dt, tau=a.tau, n_gpus=G, gpu_index=rank, device=local,
                        activation_enabled=bool(a.alpha), staleness_bound=a.tau, version_ring=a.T,
                        grace_us=a.grace_us, timeout_s=20.0)
    cfg = OptimizerConfig(T=a.T, S=a.S, tau=a.tau, alpha=bool(a.alpha), beta=not a.alpha,
                          eta=EtaSchedule(value=0.05), update_rule="momentum" if a.momentum else "sgd", momentum=0.9)
    w0 = (torch.randn(a.nelem, generator=torch.Generator().manual_seed(99), dtype=torch.float64) * 0.02).to(dt).to(dev)
    opt = GroupAveragingOptimizer(ctx, cfg, w0)
    pol = StragglerPolicy(a.victims, a.delay_us / 1000.0, selection_seed=5)
    grads = {}
    statuses = []
    for t in range(a.T):
        g = {r: synthetic_grad(r, t, a.nelem, dtype=dt, device=dev) for r in ctx.local_ranks}
        for r, v in g.items():
            grads[(t, r)] = v
        if set(ctx.local_ranks) & pol.victims(t, a.P):
            ctx.delay(int(a.delay_us * 1000))
        opt.step(t, g)
        if not a.save_grads:
            grads.clear()
        if not a.pipelined:
            torch.cuda.synchronize()
            statuses.append([(s.version, s.contrib_stamp, s.timely, s.activator) for s in ctx.statuses()])
    torch.cuda.synchronize()
    ctx.check()
    dist.barrier()
    from paper_2005_00124_b200.diagnostics import replica_diagnostics
    diag = replica_diagnostics(ctx, opt.W)
    out = {f"W{r}": opt.W[r].cpu().numpy() for r in ctx.local_ranks}
    out["gamma"] = np.array(diag.gamma)
    for (t, r), v in grads.items():
        out[f"g{t}_{r}"] = v.cpu().numpy()
    out["w0"] = w0.cpu().numpy()
    out["statuses"] = np.array(statuses, dtype=np.int64)
    if rank == 0:
        out["stamps"] = contribution_log(ctx, a.T, a.tau)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), **out)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
