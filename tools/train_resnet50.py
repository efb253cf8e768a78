"""ResNet-50 (torchvision, random init) trained with WAGMA-SGD on synthetic images.

torchrun --nproc-per-node N tools/train_resnet50.py [--S 2] [--steps 30] [--batch 32]
One WAGMA rank per GPU (P = N). Reports full training iterations/s (forward,
backward, fused WAGMA step) and the share of the step spent in the fused
WAGMA launch (CUDA events, max over ranks).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist
import torchvision

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_00124_b200.context import DeviceContext  # noqa: E402
from paper_2005_00124_b200.dist import max_over_ranks  # noqa: E402
from paper_2005_00124_b200.optim import EtaSchedule, OptimizerConfig  # noqa: E402
from paper_2005_00124_b200.torch_optim import WagmaSGD, flat_numel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--S", type=int, default=2)
ap.add_argument("--tau", type=int, default=10)
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--batch", type=int, default=32)
a = ap.parse_args()
rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
torch.manual_seed(1234)
model = torchvision.models.resnet50(weights=None).to(dev).to(memory_format=torch.channels_last)
n = flat_numel(p for p in model.parameters() if p.requires_grad)
S = min(a.S, world)
ctx = DeviceContext(world, S, n, tau=a.tau, n_gpus=world, gpu_index=rank, device=local)
cfg = OptimizerConfig(T=1 << 30, S=S, tau=a.tau, eta=EtaSchedule(value=0.1), update_rule="momentum", momentum=0.9)
opt = WagmaSGD(model.parameters(), ctx, cfg)
gen = torch.Generator(device=dev).manual_seed(rank)
x = torch.randn(a.batch, 3, 224, 224, device=dev, generator=gen).to(memory_format=torch.channels_last)
y = torch.randint(0, 1000, (a.batch,), device=dev, generator=gen)
lossf = torch.nn.CrossEntropyLoss()


def one():
    opt.zero_grad()
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = lossf(model(x), y)
    loss.backward()
    e0.record()
    opt.step()
    e1.record()
    return loss


for _ in range(a.warmup):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    one()
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
step_ms = 0.0
s0.record()
for _ in range(a.steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    loss = one()
    torch.cuda.synchronize()
    step_ms += e0.elapsed_time(e1)
s1.record()
torch.cuda.synchronize()
total_ms = max_over_ranks(s0.elapsed_time(s1), device=dev)
step_ms = max_over_ranks(step_ms, device=dev)
ctx.check()
if rank == 0:
    print(json.dumps({"model": "resnet50 (torchvision, random init)", "params": n, "gpus": world, "P": world,
                      "S": S, "batch_per_gpu": a.batch, "images": "synthetic 224x224", "amp": "bf16",
                      "train_iters_per_s": 1000.0 * a.steps / total_ms,
                      "wagma_step_ms": step_ms / a.steps, "wagma_share": step_ms / total_ms,
                      "final_loss": float(loss.detach())}))
ctx.close()
if world > 1:
    dist.destroy_process_group()
