"""Parity of the CUDA path (through the C ABI) with the reference / oracle.

- Reference trajectories (tests/golden/training_*.npz, produced by the
  reference's own `run_training` with stragglers): replayed on the device
  with the recorded contribution stamps forced -> fp64 final replicas are
  `np.array_equal` to the reference's; fp32 replicas are bit-exact with the
  fp32 oracle and within 1e-6 (norm-inf relative, test_acceptance.py:221)
  of the fp64 reference.
- Live wait-avoiding protocol (emulated stragglers on one GPU): the device
  decides who is timely; its contribution log fed to the oracle must
  reproduce every replica bit-exactly.
- Ragged sizes around the tile boundary, and a ResNet-50-sized run checked
  against the C oracle.
"""

import glob
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import c_oracle
from oracle import topology_oracle as otopo
from oracle import wagma_oracle as wo
from paper_2005_00124_b200 import _lib
from paper_2005_00124_b200.context import DeviceContext, DeviceProtocolFault, Job
from paper_2005_00124_b200.driver import TickSchedule, contribution_log, replay
from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig
from paper_2005_00124_b200.straggler import StragglerPolicy
from paper_2005_00124_b200.topology import InvalidParamsError

pytestmark = pytest.mark.gpu


def _training_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "training_*.npz")))


def _run_replay(z, meta, dtype):
    P, S, T = meta["P"], meta["S"], meta["T"]
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    ctx = DeviceContext(P, S, meta["d"], dtype=tdt, tau=meta["tau"], mask_rule=meta["mask_rule"],
                        activation_enabled=meta["alpha"] or not meta["beta"], timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=S, tau=meta["tau"], alpha=meta["alpha"], beta=meta["beta"],
                          eta=EtaSchedule(value=1.0), update_rule=meta["update_rule"], momentum=meta["momentum"])
    opt = GroupAveragingOptimizer(ctx, cfg, torch.as_tensor(z["w0"]).cuda())
    grads = torch.as_tensor(z["grads"], dtype=tdt).cuda()
    replay(opt, lambda r, t: grads[t, r], T, stamps=z["stamps"], etas=z["etas"])
    torch.cuda.synchronize()
    ctx.check()
    out = np.stack([opt.W[r].cpu().numpy() for r in range(P)])
    ctx.close()
    return out


@pytest.mark.parametrize("path", _training_cases(), ids=lambda p: os.path.basename(p)[9:-4])
def test_reference_trajectory_fp64_bit_exact(cuda, path):
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    got = _run_replay(z, meta, np.float64)
    assert np.array_equal(got, z["final"]), np.max(np.abs(got - z["final"]))


@pytest.mark.parametrize("path", _training_cases(), ids=lambda p: os.path.basename(p)[9:-4])
def test_reference_trajectory_fp32_within_1e6(cuda, path):
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    got = _run_replay(z, meta, np.float32)
    want32 = wo.replay_training(P=meta["P"], S=meta["S"], tau=meta["tau"], T=meta["T"], w0=z["w0"],
                                grads=z["grads"], etas=z["etas"], stamps=z["stamps"], alpha=meta["alpha"],
                                beta=meta["beta"], update_rule=meta["update_rule"], momentum=meta["momentum"],
                                mask_rule=meta["mask_rule"], dtype=np.float32)
    assert np.array_equal(got, want32)
    assert wo.rel_err_inf(got, z["final"]) <= 1e-6


LIVE_CASES = [
    # P, S, tau, T, n, rule, momentum, victims/iter, delay_ticks
    (8, 4, 4, 12, 10007, "example", True, 2, 1),
    (8, 2, 5, 15, 4099, "example", False, 1, 2),
    (8, 8, 10, 12, 6000, "example", True, 3, 1),
    (4, 2, 3, 10, 2048, "literal", True, 1, 1),
    (8, 4, 6, 14, 8193, "literal", False, 2, 2),
    (2, 2, 2, 6, 17, "example", True, 1, 1),
    (8, 1, 4, 8, 5000, "example", True, 2, 1),
]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("P,S,tau,T,n,rule,momentum,k,dt", LIVE_CASES)
def test_live_protocol_matches_oracle(cuda, dtype, P, S, tau, T, n, rule, momentum, k, dt):
    g = torch.Generator().manual_seed(P * 1000 + S * 10 + T)
    grads = torch.randn(T, P, n, generator=g, dtype=torch.float64) * 0.01
    w0 = torch.randn(n, generator=g, dtype=torch.float64) * 0.02
    ctx = DeviceContext(P, S, n, dtype=dtype, tau=tau, mask_rule=rule, version_ring=T, staleness_bound=tau,
                        timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=S, tau=tau, alpha=True, eta=EtaSchedule(value=0.05),
                          update_rule="momentum" if momentum else "sgd", momentum=0.9)
    opt = GroupAveragingOptimizer(ctx, cfg, w0.to(dtype).cuda())
    dg = grads.to(dtype).cuda()
    pol = StragglerPolicy(k, 1.0, selection_seed=P + T)
    TickSchedule(P, T, tau, lambda t: pol.victims(t, P), delay_ticks=dt).run(opt, lambda r, t: dg[t, r])
    torch.cuda.synchronize()
    ctx.check()
    stamps = contribution_log(ctx, T, tau)
    npdt = np.float32 if dtype == torch.float32 else np.float64
    want = wo.replay_training(P=P, S=S, tau=tau, T=T, w0=w0.numpy().astype(npdt),
                              grads=grads.numpy().astype(npdt), etas=np.full((T, P), 0.05), stamps=stamps,
                              update_rule="momentum" if momentum else "sgd", momentum=0.9, mask_rule=rule,
                              dtype=npdt)
    got = np.stack([opt.W[r].cpu().numpy() for r in range(P)])
    assert np.array_equal(got, want)
    # protocol invariants: every group version locked exactly once for all
    # ranks, ages within the staleness bound, stragglers really were stale
    for v in range(T):
        if (v + 1) % tau == 0:
            assert (stamps[v] == -2).all()
        else:
            assert (stamps[v] >= -1).all() and (stamps[v] <= v).all()
            assert (v - stamps[v]).max() <= tau - 1
    if k and P > 1:
        assert (stamps[stamps >= -1] != np.broadcast_to(np.arange(T)[:, None], stamps.shape)[stamps >= -1]).any()
    ctx.close()


@pytest.mark.parametrize("n", [1, 3, 4, 5, 2047, 2048, 2049, 6143, 3 * 2048 + 1])
def test_ragged_sizes(cuda, n):
    P, S, tau, T = 4, 2, 3, 6
    g = torch.Generator().manual_seed(n)
    grads = torch.randn(T, P, n, generator=g) * 0.1
    w0 = torch.randn(n, generator=g)
    ctx = DeviceContext(P, S, n, tau=tau, version_ring=T, timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=S, tau=tau, eta=EtaSchedule(value=0.1), update_rule="momentum")
    opt = GroupAveragingOptimizer(ctx, cfg, w0.cuda())
    dg = grads.cuda()
    pol = StragglerPolicy(1, 1.0, selection_seed=3)
    TickSchedule(P, T, tau, lambda t: pol.victims(t, P)).run(opt, lambda r, t: dg[t, r])
    torch.cuda.synchronize()
    ctx.check()
    want = wo.replay_training(P=P, S=S, tau=tau, T=T, w0=w0.numpy(), grads=grads.numpy(),
                              etas=np.full((T, P), 0.1), stamps=contribution_log(ctx, T, tau),
                              update_rule="momentum", momentum=0.9, dtype=np.float32)
    assert np.array_equal(np.stack([opt.W[r].cpu().numpy() for r in range(P)]), want)
    ctx.close()


@pytest.mark.parametrize("S", [8, 4])
def test_resnet50_sized_against_c_oracle(cuda, S):
    """N = 25,559,081 fp32, P = 8 ranks, 3 iterations incl. a global sync."""
    P, n, tau, T = 8, 25_559_081, 3, 3
    eta, beta = 0.1, 0.9
    gen = torch.Generator(device="cuda").manual_seed(1234)
    w0 = torch.randn(n, generator=gen, device="cuda") * 0.02
    ctx = DeviceContext(P, S, n, tau=tau, timeout_s=10.0)
    cfg = OptimizerConfig(T=T, S=S, tau=tau, eta=EtaSchedule(value=eta), update_rule="momentum", momentum=beta)
    opt = GroupAveragingOptimizer(ctx, cfg, w0)
    Wc = [w0.cpu().numpy().copy() for _ in range(P)]
    mc = [np.zeros(n, np.float32) for _ in range(P)]
    wp = [np.empty(n, np.float32) for _ in range(P)]
    for t in range(T):
        grads = {r: torch.randn(n, generator=gen, device="cuda") * 0.01 for r in range(P)}
        opt.step(t, grads)
        gh = [grads[r].cpu().numpy() for r in range(P)]
        sync = (t + 1) % tau == 0
        masks = [1 << j for j in range(3)] if sync else list(otopo.phase_masks(P, S, t))
        c_oracle.wagma_iteration(Wc, mc, gh, wp, masks, P if sync else S, eta, beta, True)
    torch.cuda.synchronize()
    ctx.check()
    for r in range(P):
        assert np.array_equal(opt.W[r].cpu().numpy(), Wc[r]), r
        assert np.array_equal(opt.m[r].cpu().numpy(), mc[r]), r
    ctx.close()


def test_staleness_bound_fault(cuda):
    """A rank that falls tau iterations behind trips the staleness bound
    (collective.py:290-294) -> ProtocolFault latched on the device."""
    P, S, n, T = 4, 2, 512, 8
    ctx = DeviceContext(P, S, n, tau=None, staleness_bound=2, version_ring=16, timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=S, tau=None, eta=EtaSchedule(value=0.1))
    opt = GroupAveragingOptimizer(ctx, cfg, torch.zeros(n, device="cuda"))
    g = torch.ones(n, device="cuda")
    sched = TickSchedule(P, T, None, lambda t: frozenset({1}), delay_ticks=2)
    with pytest.raises(DeviceProtocolFault) as ei:
        for versions in sched.ticks():
            opt.step_mixed(versions, {r: g for r in versions})
            torch.cuda.synchronize()
            ctx.check()
    assert ei.value.code == _lib.WG_ESTALE
    ctx.close()


def test_launch_validation(cuda):
    P, S, n = 4, 2, 64
    ctx = DeviceContext(P, S, n, tau=4, timeout_s=2.0)
    W = torch.zeros(n, device="cuda")
    g = torch.zeros(n, device="cuda")
    with pytest.raises(InvalidParamsError):  # two jobs for one rank
        ctx.launch([Job(0, _lib.WG_JOB_STEP, 0, W=W, g=g), Job(0, _lib.WG_JOB_STEP, 0, W=W, g=g)])
    with pytest.raises(InvalidParamsError):  # sync needs every local rank
        ctx.launch([Job(0, _lib.WG_JOB_SYNC_STEP, 3, W=W, g=g)])
    with pytest.raises(InvalidParamsError):  # wrong dtype / size
        ctx.launch([Job(0, _lib.WG_JOB_STEP, 0, W=torch.zeros(n + 1, device="cuda"), g=g)])
    ctx.close()


def test_replica_diagnostics(cuda):
    """Gamma_t and the post-sync bit-identity check (optim.py:199-210, 289-293)."""
    from paper_2005_00124_b200.collective import ProtocolFault
    from paper_2005_00124_b200.diagnostics import check_after_sync, gamma_bound, replica_diagnostics
    P, S, n, tau, T = 4, 2, 3001, 3, 6
    ctx = DeviceContext(P, S, n, tau=tau, timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=S, tau=tau, eta=EtaSchedule(value=0.1), update_rule="momentum")
    opt = GroupAveragingOptimizer(ctx, cfg, torch.randn(n, device="cuda"))
    g = torch.Generator(device="cuda").manual_seed(3)
    for t in range(T):
        opt.step(t, {r: torch.randn(n, device="cuda", generator=g) for r in range(P)})
        torch.cuda.synchronize()
        d = replica_diagnostics(ctx, opt.W)
        W = np.stack([opt.W[r].cpu().numpy().astype(np.float64) for r in range(P)])
        mu = W.mean(axis=0)
        assert np.allclose(d.mu.cpu().numpy(), mu, rtol=0, atol=1e-12)
        assert d.gamma == pytest.approx(float(((W - mu) ** 2).sum()), rel=1e-9)
        assert d.identical == ((t + 1) % tau == 0)  # bit-identical exactly after each global sync
        if d.identical:
            check_after_sync(d, t)
        else:
            with pytest.raises(ProtocolFault):
                check_after_sync(d, t)
    assert gamma_bound(8, 0.1, 2.0, 10) == pytest.approx(16 * 8 * 0.01 * 4 * 100)
    ctx.close()
