"""Per-iteration metrics rows on the device against the reference's recorder.

The reference's `_Recorder` (optim.py:253-307) emits one `MetricsRecord` per
iteration. Three of the golden `run_training` trajectories are replayed on
the device (fp64, contribution stamps forced from the reference's log) with
a `MetricsRecorder`; its rows must match the reference's
(tests/golden/metrics_*.npz): iteration and max_staleness exactly, gamma,
loss_mu and grad_norm_sq_mu to fp64 rounding (the device reduces in a
different order). The loss/gradient callbacks restate the reference
problems' formulas (problems.py:96-101, 149-156) on the golden problem data.
"""

import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2005_00124_b200.context import DeviceContext
from paper_2005_00124_b200.driver import replay
from paper_2005_00124_b200.metrics import CSV_HEADER, MetricsRecorder, write_run
from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig

pytestmark = pytest.mark.gpu

CASES = ["logistic_p8s4_straggle", "quad_momentum_p8s2", "quad_s8_tau8"]


def problem_fns(mz):
    prob = json.loads(str(mz["problem"]))
    if prob["kind"] == "quadratic":
        eigs, xs = mz["eigs"], mz["x_star"]

        def loss(w):
            r = w - xs
            return float(0.5 * np.dot(eigs * r, r))

        def grad(w):
            return eigs * (w - xs)
    else:
        X, y, l2 = mz["X"], mz["y"], float(mz["l2"])

        def loss(w):
            z = y * (X @ w)
            return float(np.mean(np.logaddexp(0.0, -z)) + 0.5 * l2 * np.dot(w, w))

        def grad(w):
            z = y * (X @ w)
            sig = 1.0 / (1.0 + np.exp(z))
            return -(X.T @ (y * sig)) / X.shape[0] + l2 * w
    return loss, grad


@pytest.mark.parametrize("name", CASES)
def test_metrics_rows_match_reference(cuda, tmp_path, name):
    z = np.load(os.path.join(GOLDEN, f"training_{name}.npz"))
    mz = np.load(os.path.join(GOLDEN, f"metrics_{name}.npz"))
    meta = json.loads(str(z["meta"]))
    P, S, T = meta["P"], meta["S"], meta["T"]
    ctx = DeviceContext(P, S, meta["d"], dtype=torch.float64, tau=meta["tau"], mask_rule=meta["mask_rule"],
                        timeout_s=5.0)
    cfg = OptimizerConfig(T=T, S=S, tau=meta["tau"], alpha=meta["alpha"], beta=meta["beta"],
                          eta=EtaSchedule(value=1.0), update_rule=meta["update_rule"], momentum=meta["momentum"])
    opt = GroupAveragingOptimizer(ctx, cfg, torch.as_tensor(z["w0"]).cuda())
    loss, grad = problem_fns(mz)
    rec = MetricsRecorder(opt, loss_fn=loss, grad_fn=grad)
    grads = torch.as_tensor(z["grads"]).cuda()
    replay(opt, lambda r, t: grads[t, r], T, stamps=z["stamps"], etas=z["etas"], on_step=rec.record)
    got = rec.records
    assert [r.iteration for r in got] == list(mz["iteration"])
    assert [r.max_staleness for r in got] == list(mz["max_staleness"])
    assert rec.max_staleness == meta["max_staleness"]
    np.testing.assert_allclose([r.gamma for r in got], mz["gamma"], rtol=1e-9, atol=1e-300)
    np.testing.assert_allclose([r.loss_mu for r in got], mz["loss_mu"], rtol=1e-12)
    np.testing.assert_allclose([r.grad_norm_sq_mu for r in got], mz["grad_norm_sq_mu"], rtol=1e-9)
    assert [ok for _, ok in rec.sync_replica_checks] == meta["sync_ok"]
    metrics_path, manifest_path, digest = write_run(rec, tmp_path, {"P": P, "S": S, "name": name}, seed=0)
    lines = metrics_path.read_text().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == T + 1
    man = json.loads(manifest_path.read_text())
    assert man["metrics_rows"] == T and man["metrics_sha256"] == digest and man["schema_version"] == 1
    ctx.close()
