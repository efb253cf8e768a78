"""Multi-GPU parity: one process per GPU, send rings mapped over NVLink (CUDA IPC).

Runs tests/multigpu_worker.py under torchrun on 2 or 4 GPUs with injected
device-side stragglers and checks, against the CPU oracle fed with the
device's own contribution log, that every replica is bit-exact; plus the
protocol invariants (every version locked once for all ranks, staleness
below tau, stragglers actually stale, replicas identical after each sync).
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT
from oracle import wagma_oracle as wo

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(tmp_path, G, port, env_extra=None, **kw):
    args = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
            "--master-addr", "127.0.0.1", "--master-port", str(port),
            os.path.join(ROOT, "tests", "multigpu_worker.py"), "--out", str(tmp_path)]
    for k, v in kw.items():
        args += [f"--{k.replace('_', '-')}", str(v)]
    # small test vectors: keep the split-sum kernel in play (it is off below 8 MiB by default)
    env = dict(os.environ, WG_SPLIT_MIN_BYTES="0")
    env.update(env_extra or {})
    res = subprocess.run(args, capture_output=True, text=True, timeout=900, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(G)]


@pytest.fixture(params=["mg", "hier", "nohier"])
def hier(request):
    """Kernel family: hierarchical sums in the TMA-produce kernel (WG_MG=1),
    hierarchical sums in the split / pull kernels (WG_MG=0, "hier": partials
    reduce-scattered by the split kernel where that pays, else pulled), or no
    hierarchy (split / pull kernels over the leaves, WG_HIER=0); "hier" is the default."""
    return {"mg": {"WG_HIER": "1", "WG_MG": "1"}, "hier": {"WG_HIER": "1", "WG_MG": "0"},
            "nohier": {"WG_HIER": "0", "WG_MG": "1"}}[request.param]


CASES = [
    # G, P, S, T, tau, n, dtype, victims, alpha
    (2, 2, 2, 24, 6, 10007, "f32", 1, 1),
    (2, 8, 4, 20, 5, 8192 * 3 + 5, "f32", 2, 1),
    (2, 4, 4, 16, 4, 4099, "f64", 1, 1),
    (2, 4, 2, 12, 4, 5000, "f32", 0, 0),   # blocking (beta) group allreduce
    (4, 4, 4, 20, 5, 10007, "f32", 1, 1),
    (4, 8, 8, 16, 4, 6000, "f32", 2, 1),
    (4, 8, 2, 20, 10, 4097, "f64", 2, 1),
]


@pytest.mark.parametrize("G,P,S,T,tau,n,dtype,victims,alpha", CASES)
def test_multigpu_live_protocol_bit_exact(tmp_path, hier, G, P, S, T, tau, n, dtype, victims, alpha):
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    port = 29400 + (hash((G, P, S, T, n, hier["WG_HIER"], hier["WG_MG"])) % 500)
    outs = _run(tmp_path, G, port, env_extra=hier, P=P, S=S, T=T, tau=tau, nelem=n, dtype=dtype, victims=victims,
                alpha=alpha)
    R = P // G
    npdt = np.float32 if dtype == "f32" else np.float64
    W = np.stack([outs[r // R][f"W{r}"] for r in range(P)])
    grads = np.stack([np.stack([outs[r // R][f"g{t}_{r}"] for r in range(P)]) for t in range(T)])
    w0 = outs[0]["w0"]
    if alpha:
        stamps = outs[0]["stamps"]
    else:
        stamps = np.array([[(-2 if (t + 1) % tau == 0 else t)] * P for t in range(T)], dtype=np.int64)
    want = wo.replay_training(P=P, S=S, tau=tau, T=T, w0=w0, grads=grads, etas=np.full((T, P), 0.05),
                              stamps=stamps, alpha=bool(alpha), beta=not alpha, update_rule="momentum",
                              momentum=0.9, dtype=npdt)
    assert np.array_equal(W, want)
    # device spread potential Gamma (all-reduced across the GPUs) vs numpy
    W64 = W.astype(np.float64)
    gamma = float(((W64 - W64.mean(axis=0)) ** 2).sum())
    assert float(outs[0]["gamma"]) == pytest.approx(gamma, rel=1e-9)
    if alpha:
        for v in range(T):
            if (v + 1) % tau == 0:
                continue
            assert (stamps[v] >= -1).all() and (stamps[v] <= v).all(), (v, stamps[v])
            assert (v - stamps[v]).max() <= tau - 1
        if victims:
            late = sum(int((stamps[v] >= -1).sum() - (stamps[v] == v).sum()) for v in range(T))
            assert late > 0, "injected stragglers never contributed a stale model"


BASELINE_CASES = [
    # G, S: P = 8 ranks, n = 25,559,081 fp32 (BASELINE configs[1]), tau = 10, T = 12 (one global sync)
    (2, 8), (2, 4), (4, 8), (4, 4),
]


def _replay_streaming(P, S, tau, T, n, w0, grad_fn, stamps, eta=0.05, beta=0.9):
    """Alg. 2 for all P ranks with the C oracle, holding only the send-buffer
    snapshots the contribution log references (BASELINE-sized vectors)."""
    from oracle import c_oracle
    from oracle import topology_oracle as otopo
    W = [w0.copy() for _ in range(P)]
    m = [np.zeros(n, np.float32) for _ in range(P)]
    wp = [np.empty(n, np.float32) for _ in range(P)]
    keep = {(q, int(s)) for v in range(T) for q, s in enumerate(stamps[v]) if 0 <= s < v}
    needs_w0 = bool((stamps == -1).any())
    sendbuf = {(q, -1): w0 for q in range(P)} if needs_w0 else {}
    for t in range(T):
        g = [grad_fn(r, t) for r in range(P)]
        sync = (t + 1) % tau == 0
        if sync:
            masks, div, contrib, timely = [1 << j for j in range(P.bit_length() - 1)], P, None, None
        else:
            masks, div = list(otopo.phase_masks(P, S, t)), S
            contrib = [None if int(stamps[t, q]) == t else sendbuf[(q, int(stamps[t, q]))] for q in range(P)]
            timely = [int(stamps[t, q]) == t for q in range(P)]
        c_oracle.wagma_iteration(W, m, g, wp, masks, div, eta, beta, True, contrib=contrib, timely=timely)
        for q in range(P):
            if (q, t) in keep:
                sendbuf[(q, t)] = wp[q].copy()
    return np.stack(W)


@pytest.mark.parametrize("G,S", BASELINE_CASES)
def test_multigpu_baseline_size_bit_exact(tmp_path, hier, G, S):
    """BASELINE configs[1] on 2 / 4 GPUs: P = 8, n = 25,559,081, one straggler GPU
    per iteration, launches pipelined as in bench.py, default split threshold;
    every replica bit-exact against the C oracle fed the device contribution log."""
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    import torch

    from paper_2005_00124_b200.driver import synthetic_grad
    P, T, tau, n = 8, 12, 10, 25_559_081
    port = 29950 + (hash((G, S, hier["WG_HIER"], hier["WG_MG"])) % 40)
    env = dict(hier, WG_SPLIT_MIN_BYTES=str(8 << 20))
    outs = _run(tmp_path, G, port, env_extra=env, P=P, S=S, T=T, tau=tau, nelem=n, dtype="f32", victims=1,
                pipelined=1, save_grads=0, delay_us=300)
    R = P // G
    Wdev = np.stack([outs[r // R][f"W{r}"] for r in range(P)])
    stamps = outs[0]["stamps"]
    w0 = outs[0]["w0"]

    def grad_fn(r, t):
        return synthetic_grad(r, t, n, dtype=torch.float32, device="cuda").cpu().numpy()

    want = _replay_streaming(P, S, tau, T, n, w0, grad_fn, stamps)
    assert np.array_equal(Wdev, want)
    late = sum(int((stamps[v] >= -1).sum() - (stamps[v] == v).sum()) for v in range(T) if (v + 1) % tau)
    assert late > 0, "the injected straggler never contributed a stale model"


def test_multigpu_mismatched_sync_points():
    """collective.py:381-386 on the device: rank 0 (GPU 0) joins iteration 0 as
    a global sync, rank 1 (GPU 1) as a group round; both GPUs latch WG_ESYNC
    (ProtocolFault) instead of a watchdog timeout."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    args = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
            "--master-addr", "127.0.0.1", "--master-port", "29391",
            os.path.join(ROOT, "tests", "sync_mismatch_worker.py")]
    res = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "rank0 code=9" in res.stdout and "rank1 code=9" in res.stdout


STRESS_CASES = [
    # G, P, S, families: default kernels (split / pull, GPU-scope flag fences) and the hierarchical ones
    (2, 8, 8), (4, 8, 8), (4, 8, 4), (4, 4, 2),
]


@pytest.mark.parametrize("G,P,S", STRESS_CASES)
def test_multigpu_stress_pipelined_rounds(tmp_path, hier, G, P, S):
    """Memory-model stress (the default GPU-scope flag fences rely
    on peers' loads being served by the owner's L2): 300 pipelined iterations
    (no host synchronisation between launches), a rotating straggler GPU,
    ragged n of a few chunks so flag publication and consumption race on every
    tile; every replica must stay bit-exact against the oracle."""
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    T, tau, n = 300, 10, 3 * 2048 + 7
    port = 29700 + (hash((G, P, S, hier["WG_HIER"], hier["WG_MG"])) % 200)
    outs = _run(tmp_path, G, port, env_extra=hier, P=P, S=S, T=T, tau=tau, nelem=n, dtype="f32", victims=1,
                pipelined=1, delay_us=40)
    R = P // G
    W = np.stack([outs[r // R][f"W{r}"] for r in range(P)])
    grads = np.stack([np.stack([outs[r // R][f"g{t}_{r}"] for r in range(P)]) for t in range(T)])
    stamps = outs[0]["stamps"]
    want = wo.replay_training(P=P, S=S, tau=tau, T=T, w0=outs[0]["w0"], grads=grads, etas=np.full((T, P), 0.05),
                              stamps=stamps, update_rule="momentum", momentum=0.9, dtype=np.float32)
    assert np.array_equal(W, want)
    late = sum(int((stamps[v] >= -1).sum() - (stamps[v] == v).sum()) for v in range(T) if (v + 1) % tau)
    assert late > 0, "the rotating straggler never contributed a stale model"
