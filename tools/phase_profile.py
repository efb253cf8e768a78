"""Per-CTA phase breakdown of the multi-GPU step kernel (device clock64 counters).

torchrun --nproc-per-node N tools/phase_profile.py [--S 8] [--P 8] [--n N]
Prints, per rank, the mean over CTAs of cycles spent producing, publishing
(barrier + system fence + flags), resolving sources, polling peer flags and
consuming, for a group step and a sync step.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_00124_b200.context import DeviceContext  # noqa: E402
from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--S", type=int, default=8)
ap.add_argument("--nelem", type=int, default=25_559_081)
ap.add_argument("--tau", type=int, default=10)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--S2", type=int, default=0)
a = ap.parse_args()
rank, G, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ctx = DeviceContext(a.P, a.S, a.nelem, tau=a.tau, n_gpus=G, gpu_index=rank, device=local)
opt = GroupAveragingOptimizer(ctx, OptimizerConfig(T=1 << 30, S=a.S, tau=a.tau, eta=EtaSchedule(value=0.1),
                                                   update_rule="momentum"), torch.zeros(a.nelem, device=dev))
g = {r: torch.randn(a.nelem, device=dev) * 0.01 for r in ctx.local_ranks}
prof = torch.zeros(max(ctx.grid, ctx.lib_sms if hasattr(ctx, "lib_sms") else 148) * 16, dtype=torch.int64,
                   device=dev)
ctx.lib.wg_ctx_set_profile(ctx._h, ctypes.c_void_p(prof.data_ptr()))
ghz = 1.965
for t in range(a.iters):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()  # start the 8 launches together (skew > grace window makes a GPU stale)
    for u in range(8):  # back to back (steady state), profile the last launch
        if u == 7:
            prof.zero_()
            ev0.record()
        opt.step(t * 8 + u, g)
    ev1.record()
    torch.cuda.synchronize()
    t = t * 8 + 7
    if True:
        split_prof = os.environ.get("WG_PROF_SPLIT", "0") == "1" or os.environ.get("WG_PROF_MG", "0") == "1"
        p = prof.view(-1, 16 if split_prof else 8).cpu().numpy().astype(np.float64)
        if os.environ.get("WG_PROF_MG", "0") == "1":
            names = ["cons_total", "cons_in_wait", "cons_ph1_wait", "cons_ack_wait", "cons_ready_wait",
                     "pullA_poll", "pullA_empty", "pullA_total", "pub_wait", "pub_fence", "pub_total",
                     "ready_at", "prod_empty_wait", "prod_total", "x", "x"]
        elif os.environ.get("WG_PROF_SPLIT", "0") == "1":
            names = ["producer_total", "pullA_total", "x", "redA_full_wait", "redA_total", "pullB_total", "finB_full_wait", "finB_total", "pullA_empty", "pullA_poll", "x", "pullB_empty", "pullB_poll", "x", "fin_ready_at", "fin_work"]
        elif os.environ.get("WG_NVL", "1") != "0":
            names = ["producer_total", "pull_empty_wait", "pull_poll", "pull_issue", "cons_full_wait", "x", "cons_total", "cons_ready_wait"]
        else:
            names = ["produce", "publish", "resolve", "poll", "consume", "tiles", "fence"]
        us = {nm: p[:, i].mean() / ghz / 1000 for i, nm in enumerate(names) if nm not in ("tiles", "x")}
        sync = (t + 1) % a.tau == 0
        if os.environ.get("WG_PROF_DUMP"):
            np.save(f"{os.environ['WG_PROF_DUMP']}_r{rank}_t{t}.npy", p)
        mx = {nm: p[:, i].max() / ghz / 1000 for i, nm in enumerate(names) if nm not in ("tiles", "x")}
        stamps, locked = ctx.query_version(t) if not sync else ([t] * a.P, True)
        stale = sum(1 for x in stamps if x != t)
        print(f"rank{rank} t={t} stale={stale} {'sync ' if sync else 'group'} kernel={ev0.elapsed_time(ev1)*1000:.0f}us "
              + " ".join(f"{k}={v:.0f}/{mx[k]:.0f}" for k, v in us.items()), flush=True)
ctx.lib.wg_ctx_set_profile(ctx._h, None)
ctx.check()
dist.barrier()
dist.destroy_process_group()
