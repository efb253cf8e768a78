"""`torch.optim.Optimizer` front end: WAGMA-SGD over a model's flattened parameters.

The step before the hot path: instead of a problem's
gradient oracle (`local_step`, optim.py:172-173), gradients come from
autograd on a real model. The model's parameters are re-pointed into one
flat, 16-byte aligned fp32 buffer (the replica W the fused kernel updates in
place) and their `.grad` into a flat gradient buffer that autograd
accumulates into, so `optimizer.step()` is exactly one fused device launch:
momentum step, send-ring install, wait-avoiding group average over NVLink.

One WAGMA rank per process (one replica per GPU); run under torchrun with
`DeviceContext(P=world, ..., n_gpus=world, gpu_index=rank)`.
"""

from __future__ import annotations

from typing import Iterable, Optional

import torch

from .context import DeviceContext
from .optim import GroupAveragingOptimizer, OptimizerConfig

__all__ = ["WagmaSGD", "flat_numel"]


def flat_numel(params: Iterable[torch.nn.Parameter]) -> int:
    return sum(p.numel() for p in params)


class WagmaSGD(torch.optim.Optimizer):
    """WAGMA-SGD (Alg. 2 of arXiv 2005.00124) as a torch optimizer.

    ``cfg`` carries eta / momentum / S / tau / alpha / beta exactly like the
    reference's `OptimizerConfig` (optim.py:106-148); the context must host
    exactly one rank. Model buffers (e.g. BatchNorm statistics) stay local.
    """

    def __init__(self, params: Iterable[torch.nn.Parameter], ctx: DeviceContext, cfg: OptimizerConfig):
        params = [p for p in params if p.requires_grad]
        if len(ctx.local_ranks) != 1:
            raise ValueError("WagmaSGD drives one WAGMA rank per process")
        n = flat_numel(params)
        if n != ctx.n:
            raise ValueError(f"context was created for n={ctx.n} elements, the parameters have {n}")
        super().__init__(params, dict(lr=cfg.eta.value))
        self.ctx = ctx
        self.cfg = cfg
        self.rank = ctx.local_ranks[0]
        dev = ctx.torch_device
        self.flat = torch.zeros(n, dtype=ctx.dtype, device=dev)
        self.flat_grad = torch.zeros(n, dtype=ctx.dtype, device=dev)
        off = 0
        with torch.no_grad():
            for p in params:
                k = p.numel()
                self.flat[off:off + k].copy_(p.detach().reshape(-1))
                p.data = self.flat[off:off + k].view_as(p)
                p.grad = self.flat_grad[off:off + k].view_as(p)
                off += k
        self._params = params
        # every rank starts from the same initial point (optim.py:328): rank 0's
        if ctx.n_gpus > 1:
            import torch.distributed as dist
            dist.broadcast(self.flat, src=0)
        self.engine = GroupAveragingOptimizer(ctx, cfg, self.flat)
        # the engine owns the replica tensor W[rank]: make it the parameters' storage
        self.engine.W[self.rank] = self.flat
        self.iteration = 0

    def zero_grad(self, set_to_none: bool = False) -> None:  # keep the flat .grad views
        self.flat_grad.zero_()

    @torch.no_grad()
    def step(self, closure: Optional[callable] = None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        for p in self._params:  # autograd must have accumulated into the flat views
            if p.grad is None or p.grad.data_ptr() < self.flat_grad.data_ptr() or \
                    p.grad.data_ptr() >= self.flat_grad.data_ptr() + self.flat_grad.numel() * self.flat_grad.element_size():
                raise RuntimeError("parameter .grad was replaced; call zero_grad() (not set_to_none)")
        self.engine.step(self.iteration, {self.rank: self.flat_grad})
        self.iteration += 1
        return loss
