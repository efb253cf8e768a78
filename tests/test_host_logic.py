"""Host-side logic of the drop-in modules (CPU only).

StragglerPolicy / compute_delay against the reference's own victim draws
(tests/golden/topology.json), the new length-bucket delay model, the
configuration API restated from the reference's optimizer tests
(`pkg/tests/test_optim.py:103-161`), and the launch-tick straggler emulation.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2005_00124_b200.driver import TickSchedule
from paper_2005_00124_b200.optim import ConfigError, EtaSchedule, OptimizerConfig, is_sync_iteration
from paper_2005_00124_b200.straggler import (
    BucketedLengthDelay,
    DelayModel,
    StragglerPolicy,
    compute_delay,
)


def test_victims_match_reference():
    with open(os.path.join(GOLDEN, "topology.json")) as fp:
        golden = json.load(fp)["victims"]
    for seed, P, k, t, want in golden:
        assert sorted(StragglerPolicy(k, 1.0, selection_seed=seed).victims(t, P)) == want


def test_compute_delay_rules():
    pol = StragglerPolicy(2, 320.0, selection_seed=3)
    dm = DelayModel(base_compute_ms=100.0, jitter_max_ms=5.0, straggler=pol)
    for t in range(6):
        vict = pol.victims(t, 8)
        for r in range(8):
            d = compute_delay(r, t, dm, 11, 8)
            assert d == compute_delay(r, t, dm, 11, 8)  # pure
            extra = 320.0 if r in vict else 0.0
            assert 100.0 + extra <= d <= 105.0 + extra
    with pytest.raises(ValueError):
        compute_delay(8, 0, dm, 11, 8)
    with pytest.raises(ValueError):
        StragglerPolicy(9, 1.0).victims(0, 8)
    with pytest.raises(ValueError):
        DelayModel(base_compute_ms=-1.0)


def test_bucketed_length_delay():
    d = BucketedLengthDelay(2.0, seed=7)
    draws = np.array([d.delay_ms(r, t) for t in range(400) for r in range(8)])
    assert draws.min() > 0 and draws.max() <= 2.0 * 256 / d.mean_length() + 1e-12
    assert abs(draws.mean() - 2.0) < 0.15  # mean compute time = base
    assert d.delay_ms(3, 5) == BucketedLengthDelay(2.0, seed=7).delay_ms(3, 5)
    assert len({round(x, 9) for x in draws}) > 3  # actually imbalanced


def test_eta_and_config_known_answers():
    sched = EtaSchedule(kind="step", value=0.8, decay_factor=0.5, decay_every=3)
    assert [sched.rate(t, 4, 100) for t in (0, 2, 3, 6)] == [0.8, 0.8, 0.4, 0.2]
    assert EtaSchedule(kind="theorem").rate(0, 16, 400) == 16 / 20.0
    with pytest.raises(ConfigError):
        EtaSchedule(kind="cosine").rate(0, 1, 1)
    with pytest.raises(ConfigError):
        EtaSchedule(kind="step", decay_every=0).rate(0, 1, 1)
    for bad in (dict(alpha=True, beta=True), dict(T=0), dict(tau=0), dict(b=0), dict(update_rule="adam"),
                dict(S=3), dict(S=16)):
        kw = dict(T=10, S=4, tau=5)
        kw.update(bad)
        with pytest.raises(ConfigError):
            OptimizerConfig(**kw).validate(8)
    with pytest.raises(ConfigError):
        OptimizerConfig(T=10, eta=EtaSchedule(value=0.0)).validate(8)
    OptimizerConfig(T=10, S=4, tau=5).validate(8)
    assert [t for t in range(12) if is_sync_iteration(t, 4)] == [3, 7, 11]
    assert not is_sync_iteration(3, None)


@pytest.mark.parametrize("P,T,tau,k,dt", [(8, 20, 5, 2, 1), (4, 17, 4, 1, 2), (8, 12, None, 1, 1)])
def test_tick_schedule_properties(P, T, tau, k, dt):
    pol = StragglerPolicy(k, 1.0, selection_seed=5)
    sched = TickSchedule(P, T, tau, lambda t: pol.victims(t, P), delay_ticks=dt)
    done = {r: [] for r in range(P)}
    for versions in sched.ticks():
        assert len(versions) <= P
        sync_ts = {t for t in versions.values() if is_sync_iteration(t, tau)}
        if sync_ts:  # a global sync launches all ranks together at one version
            assert len(versions) == P and len(set(versions.values())) == 1
        for r, t in versions.items():
            done[r].append(t)
    for r in range(P):
        assert done[r] == list(range(T))  # every rank runs every iteration once, in order


def test_activation_message_counts_match_reference():
    """Per-rank ACT counts of a single-root activation, against the reference's
    own endpoints on its simulator (tests/golden/activation.json)."""
    import json

    from conftest import GOLDEN
    from paper_2005_00124_b200.collective import activation_acts

    cases = json.load(open(os.path.join(GOLDEN, "activation.json")))
    assert len(cases) >= 50
    for c in cases:
        P, S, root = c["P"], c["S"], c["root"]
        assert [activation_acts(r, root, P) for r in range(P)] == c["acts_sent"], c
        assert sum(c["acts_sent"]) == P - 1
        assert c["activations_originated"] == [int(r == root) for r in range(P)]
        assert c["phases_sent"] == [S.bit_length() - 1] * P


def test_metrics_csv_format_matches_reference():
    """MetricsRecord.csv_row reproduces the reference's rows (optim.py:229-234)
    byte for byte when given the reference's values (tests/golden/metrics_*.npz)."""
    import glob
    import os

    import numpy as np

    from conftest import GOLDEN
    from paper_2005_00124_b200.metrics import CSV_HEADER, MetricsRecord

    for path in sorted(glob.glob(os.path.join(GOLDEN, "metrics_*.npz"))):
        lines = str(np.load(path)["csv"]).split("\n")
        assert lines[0] == CSV_HEADER
        for line in lines[1:]:
            f = line.split(",")
            rec = MetricsRecord(int(f[0]), float(f[1]), float(f[2]), float(f[3]), float(f[4]), int(f[5]),
                                int(f[6]), int(f[7]))
            assert rec.csv_row() == line


def test_fixed_victims_policy():
    """C4's fixed straggler (tests/test_optim.py:193-197 `_FixedVictims`)."""
    import pytest

    from paper_2005_00124_b200.straggler import FixedVictims
    pol = FixedVictims(1, 5.0)
    assert all(pol.victims(t, 4) == frozenset({1}) for t in range(20))
    assert pol.extra_delay_ms == 5.0
    with pytest.raises(ValueError):
        FixedVictims(4, 1.0).victims(0, 4)


def test_optimizer_fast_step_job_array():
    """GroupAveragingOptimizer.step's host fast path (no GPU: a stand-in context
    records the wg_job array): per-step fields follow t (kind: sync every tau,
    version, step size), fixed fields are rewritten when a replica is replaced,
    gradients are validated, misaligned gradients fall back to the general path."""
    import types

    import torch

    from paper_2005_00124_b200 import _lib
    from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig
    from paper_2005_00124_b200.topology import InvalidParamsError

    n = 64
    launched = []

    class Ctx:
        P, S, n, dtype = 4, 2, 64, torch.float32
        torch_device = torch.device("cpu")
        local_ranks = (0, 1)

        def launch_array(self, arr, k, forced, stream):
            launched.append([(arr[i].rank, arr[i].kind, arr[i].version, arr[i].eta, arr[i].W, arr[i].m, arr[i].g,
                              arr[i].beta, arr[i].update_rule) for i in range(k)])

        def _check_vec(self, t, name):
            if t is not None and (t.dtype != self.dtype or t.numel() != self.n):
                raise InvalidParamsError(name)

    ctx = Ctx()
    opt = object.__new__(GroupAveragingOptimizer)
    opt.ctx, opt.cfg, opt.T = ctx, OptimizerConfig(T=10, S=2, tau=3, eta=EtaSchedule(value=0.25),
                                                    update_rule="momentum", momentum=0.9), 10
    opt.use_group, opt.momentum = True, True
    opt.W = {r: torch.zeros(n) for r in ctx.local_ranks}
    opt.m = {r: torch.zeros(n) for r in ctx.local_ranks}
    opt._arr, opt._slot = None, []
    opt._wptr = {r: w.data_ptr() for r, w in opt.W.items()}
    opt._mptr = {r: w.data_ptr() for r, w in opt.m.items()}
    g = {r: torch.ones(n) for r in ctx.local_ranks}
    for t in range(3):
        assert opt._fast_step(t, g, None, None)
    kinds = [row[0][1] for row in launched]
    assert kinds == [_lib.WG_JOB_STEP, _lib.WG_JOB_STEP, _lib.WG_JOB_SYNC_STEP]  # (t+1) % tau == 0
    assert [row[0][2] for row in launched] == [0, 1, 2]
    r0 = launched[-1][0]
    assert r0[0] == 0 and r0[3] == 0.25 and r0[7] == 0.9 and r0[8] == _lib.WG_UPDATE_MOMENTUM
    assert r0[4] == opt.W[0].data_ptr() and r0[5] == opt.m[0].data_ptr() and r0[6] == g[0].data_ptr()
    # a replaced replica: its new pointer reaches the array
    opt.W[1] = torch.full((n,), 2.0)
    assert opt._fast_step(3, g, None, None)
    assert launched[-1][1][4] == opt.W[1].data_ptr()
    # a wrong-sized gradient is rejected; a misaligned one takes the general path
    with pytest.raises(InvalidParamsError):
        opt._fast_step(4, {0: torch.ones(n + 1)}, None, None)
    misaligned = torch.ones(n + 1)[1:]
    assert not opt._fast_step(4, {0: misaligned}, None, None)
    with pytest.raises(InvalidParamsError):  # not a rank of this process
        opt._fast_step(4, {3: torch.ones(n)}, None, None)
