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


def _run(tmp_path, G, port, **kw):
    args = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
            "--master-addr", "127.0.0.1", "--master-port", str(port),
            os.path.join(ROOT, "tests", "multigpu_worker.py"), "--out", str(tmp_path)]
    for k, v in kw.items():
        args += [f"--{k.replace('_', '-')}", str(v)]
    # small test vectors: keep the split-sum kernel in play (it is off below 8 MiB by default)
    env = dict(os.environ, WG_SPLIT_MIN_BYTES="0")
    res = subprocess.run(args, capture_output=True, text=True, timeout=600, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return [dict(np.load(os.path.join(tmp_path, f"rank{r}.npz"))) for r in range(G)]


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
def test_multigpu_live_protocol_bit_exact(tmp_path, G, P, S, T, tau, n, dtype, victims, alpha):
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs")
    port = 29400 + (hash((G, P, S, T, n)) % 500)
    outs = _run(tmp_path, G, port, P=P, S=S, T=T, tau=tau, nelem=n, dtype=dtype, victims=victims, alpha=alpha)
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
