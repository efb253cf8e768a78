"""Kernel-level GPU checks: the single-GPU TMA kernel against the cp.async
kernel and the oracle, DivergenceError, and parity at the C3/C4 sizes.

- `wagma_local_kernel` (TMA bulk-copy producer warp, default on one GPU) and
  the older per-thread cp.async kernel (`WG_LOC=0`) must both reproduce the
  oracle bit for bit on the live protocol with emulated stragglers (mixed
  versions in one launch, stale leaves read from older send slots).
- A non-finite gradient latches WG_EDIVERGE on the device; the host raises
  `DivergenceError` (optim.py:174-175) from `ctx.check()` and, without any
  synchronisation of its own, from the next `step()`.
- C4 (DD-PPO, n = 8,476,421) and C3 (Transformer-big, n = 213,000,000) sized
  runs through a global sync, bit-exact against the C oracle.
"""

import numpy as np
import pytest
import torch

from oracle import c_oracle
from oracle import topology_oracle as otopo
from oracle import wagma_oracle as wo
from paper_2005_00124_b200.context import DeviceContext, DivergenceError
from paper_2005_00124_b200.driver import TickSchedule, contribution_log
from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig
from paper_2005_00124_b200.straggler import StragglerPolicy

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["tma", "cpasync"])
def kernel(request, monkeypatch):
    """Select the single-GPU kernel for contexts created in the test (WG_LOC is read at creation)."""
    monkeypatch.setenv("WG_LOC", "1" if request.param == "tma" else "0")
    return request.param


CASES = [
    # P, S, tau, T, n, momentum, victims/iter, delay_ticks, dtype
    (8, 8, 5, 12, 25_000, True, 2, 1, torch.float32),
    (8, 4, 4, 12, 2 * 2048 + 3, True, 2, 2, torch.float32),
    (8, 2, 6, 14, 3 * 1024 + 1, False, 3, 1, torch.float32),
    (4, 4, 3, 10, 7777, True, 1, 1, torch.float64),
    (16, 4, 4, 10, 4096, True, 3, 1, torch.float32),
    (2, 1, 3, 7, 1, True, 1, 1, torch.float32),
]


@pytest.mark.parametrize("P,S,tau,T,n,momentum,k,dt,dtype", CASES)
def test_single_gpu_kernels_match_oracle(cuda, kernel, P, S, tau, T, n, momentum, k, dt, dtype):
    g = torch.Generator().manual_seed(P * 7 + S * 3 + n)
    grads = torch.randn(T, P, n, generator=g, dtype=torch.float64) * 0.01
    w0 = torch.randn(n, generator=g, dtype=torch.float64) * 0.02
    ctx = DeviceContext(P, S, n, dtype=dtype, tau=tau, version_ring=T, timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=S, tau=tau, eta=EtaSchedule(value=0.05),
                          update_rule="momentum" if momentum else "sgd", momentum=0.9)
    opt = GroupAveragingOptimizer(ctx, cfg, w0.to(dtype).cuda())
    dg = grads.to(dtype).cuda()
    pol = StragglerPolicy(k, 1.0, selection_seed=P + T + n)
    TickSchedule(P, T, tau, lambda t: pol.victims(t, P), delay_ticks=dt).run(opt, lambda r, t: dg[t, r])
    torch.cuda.synchronize()
    ctx.check()
    stamps = contribution_log(ctx, T, tau)
    npdt = np.float32 if dtype == torch.float32 else np.float64
    want = wo.replay_training(P=P, S=S, tau=tau, T=T, w0=w0.numpy().astype(npdt),
                              grads=grads.numpy().astype(npdt), etas=np.full((T, P), 0.05), stamps=stamps,
                              update_rule="momentum" if momentum else "sgd", momentum=0.9, dtype=npdt)
    got = np.stack([opt.W[r].cpu().numpy() for r in range(P)])
    assert np.array_equal(got, want)
    ctx.close()


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")], ids=["nan", "inf", "-inf"])
def test_non_finite_gradient_raises_divergence(cuda, kernel, bad):
    P, S, n, tau = 4, 2, 10_000, 4
    ctx = DeviceContext(P, S, n, tau=tau, timeout_s=5.0)
    cfg = OptimizerConfig(T=8, S=S, tau=tau, eta=EtaSchedule(value=0.1), update_rule="momentum")
    opt = GroupAveragingOptimizer(ctx, cfg, torch.zeros(n, device="cuda"))
    grads = {r: torch.full((n,), 0.01, device="cuda") for r in range(P)}
    opt.step(0, grads)
    torch.cuda.synchronize()
    ctx.check()  # finite: nothing latched
    grads[2] = grads[2].clone()
    grads[2][n - 3] = bad
    opt.step(1, grads)
    torch.cuda.synchronize()
    with pytest.raises(DivergenceError) as ei:
        ctx.check()
    assert ei.value.rank == 2
    with pytest.raises(DivergenceError):  # the next step refuses, from the mapped error word
        opt.step(2, {r: torch.zeros(n, device="cuda") for r in range(P)})
    ctx.close()


def test_divergence_check_is_per_element_not_padding(cuda, kernel):
    """Elements past n (tile padding) never count as divergent."""
    P, S, n, tau = 2, 2, 1025, 3
    ctx = DeviceContext(P, S, n, tau=tau, timeout_s=5.0)
    cfg = OptimizerConfig(T=4, S=S, tau=tau, eta=EtaSchedule(value=0.1))
    opt = GroupAveragingOptimizer(ctx, cfg, torch.zeros(n, device="cuda"))
    for t in range(4):
        opt.step(t, {r: torch.full((n,), 1e-3, device="cuda") for r in range(P)})
    torch.cuda.synchronize()
    ctx.check()
    ctx.close()


def _against_c_oracle(P, S, n, tau, T, *, seed=1234):
    eta, beta = 0.1, 0.9
    gen = torch.Generator(device="cuda").manual_seed(seed)
    w0 = torch.randn(n, generator=gen, device="cuda") * 0.02
    ctx = DeviceContext(P, S, n, tau=tau, timeout_s=20.0)
    cfg = OptimizerConfig(T=T, S=S, tau=tau, eta=EtaSchedule(value=eta), update_rule="momentum", momentum=beta)
    opt = GroupAveragingOptimizer(ctx, cfg, w0)
    Wc = [w0.cpu().numpy().copy() for _ in range(P)]
    mc = [np.zeros(n, np.float32) for _ in range(P)]
    wp = [np.empty(n, np.float32) for _ in range(P)]
    for t in range(T):
        grads = {r: torch.randn(n, generator=gen, device="cuda") * 0.01 for r in range(P)}
        opt.step(t, grads)
        gh = [grads[r].cpu().numpy() for r in range(P)]
        del grads
        sync = (t + 1) % tau == 0
        masks = [1 << j for j in range(P.bit_length() - 1)] if sync else list(otopo.phase_masks(P, S, t))
        c_oracle.wagma_iteration(Wc, mc, gh, wp, masks, P if sync else S, eta, beta, True)
    torch.cuda.synchronize()
    ctx.check()
    for r in range(P):
        assert np.array_equal(opt.W[r].cpu().numpy(), Wc[r]), r
        assert np.array_equal(opt.m[r].cpu().numpy(), mc[r]), r
    ctx.close()


@pytest.mark.parametrize("S", [8, 2])
def test_c4_ddppo_sized_against_c_oracle(cuda, kernel, S):
    """C4: N = 8,476,421 fp32, P = 8 ranks, 3 iterations (tau = 3: the third is a global sync)."""
    _against_c_oracle(8, S, 8_476_421, 3, 3)


def test_c3_transformer_big_sized_against_c_oracle(cuda):
    """C3: N = 213,000,000 fp32 (852 MB per replica), P = 4, S = 4, through a global sync."""
    _against_c_oracle(4, 4, 213_000_000, 2, 3, seed=7)
