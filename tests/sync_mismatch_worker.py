"""Two processes, one GPU each, P = 2 ranks, S = 2 (launched by torchrun from
test_gpu_multi.py): rank 0 joins iteration 0 as a global sync, rank 1 joins it
as a group round -- the reference's "mismatched sync points" fault
(collective.py:381-386). Both launches consume each other's W'_0 (nobody
hangs); each process must then see WG_ESYNC latched on its device."""

import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2005_00124_b200 import _lib  # noqa: E402
from paper_2005_00124_b200.context import DeviceContext, DeviceProtocolFault, Job  # noqa: E402


def main():
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n = 4096
    ctx = DeviceContext(2, 2, n, dtype=torch.float32, tau=4, n_gpus=2, gpu_index=rank, device=local, timeout_s=10.0)
    W = torch.zeros(n, device=dev)
    m = torch.zeros(n, device=dev)
    g = torch.ones(n, device=dev)
    kind = _lib.WG_JOB_SYNC_STEP if rank == 0 else _lib.WG_JOB_STEP
    ctx.launch([Job(rank=rank, kind=kind, version=0, W=W, m=m, g=g, eta=0.1, beta=0.9, momentum=True)])
    torch.cuda.synchronize()
    try:
        ctx.check()
        code = 0
    except DeviceProtocolFault as exc:
        code = exc.code
    dist.barrier()
    print(f"rank{rank} code={code}", flush=True)
    ctx.close()
    dist.destroy_process_group()
    sys.exit(0 if code == _lib.WG_ESYNC else 3)


if __name__ == "__main__":
    main()
