"""Host cost of one fused step launch (Python + ctypes + C++ planning), no sync."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_00124_b200.context import DeviceContext
from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig
for P, S in [(8, 8), (8, 2), (1, 1)]:
    n = 4096
    ctx = DeviceContext(P, S, n, tau=10)
    opt = GroupAveragingOptimizer(ctx, OptimizerConfig(T=1 << 30, S=S, tau=10, eta=EtaSchedule(value=0.1), update_rule="momentum"),
                                  torch.zeros(n, device="cuda"))
    g = {r: torch.randn(n, device="cuda") for r in ctx.local_ranks}
    for t in range(50):
        opt.step(t, g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K = 2000
    for t in range(50, 50 + K):
        opt.step(t, g)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    jobs = opt.jobs({r: 7 for r in ctx.local_ranks}, g)
    t3 = time.perf_counter()
    for _ in range(K):
        opt.jobs({r: 7 for r in ctx.local_ranks}, g)
    t4 = time.perf_counter()
    print(f"P={P} S={S}: host {1e6*(t1-t0)/K:.1f} us/step (jobs() alone {1e6*(t4-t3)/K:.1f} us), incl. GPU drain {1e6*(t2-t0)/K:.1f} us/step")
    ctx.close()
