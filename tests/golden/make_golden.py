"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

This script is the only thing in the repo that imports the reference
(`/root/reference/pkg/src/wagma`, pure Python + numpy). It runs in the build
container (where /root/reference exists) and writes small, committed
fixtures that the CPU and GPU parity tests read at run time, so nothing on
the GPU box ever needs the reference:

  topology.json     phase masks (both rules) on the A2 grid P<=1024
                    (`tests/test_acceptance.py:38-47`), sha256 of every
                    partition, full partitions for P<=32, mixing results,
                    peer known answers.
  collective.npz    group-round accumulators produced by the reference's
                    own `GroupAllreduce` endpoints on its `Simulator`
                    (all-timely, stale/late, literal rule, sync).
  activation.json   per-rank ACT / PHASE message counters of one version
                    activated by a single root (`collective.py:182-184`,
                    `:263-274`, `:319`) for every root, P <= 16.
  training_*.npz    `run_training` trajectories with the per-(rank, t)
                    gradients, the contribution log (rank, version, stamp)
                    captured from `optim._ContributionSink.append`
                    (`optim.py:310-319`), and the final weights.
  metrics_*.npz     the reference's per-iteration `MetricsRecord` rows
                    (`optim.py:218-234`) of three of those trajectories and
                    the problem data their loss/gradient columns need.

Usage:  python tests/golden/make_golden.py   (from the repo root)
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

REF_SRC = os.environ.get("WAGMA_REFERENCE_SRC", "/root/reference/pkg/src")
sys.dont_write_bytecode = True  # the reference tree is read-only
sys.path.insert(0, REF_SRC)

from wagma import collective as ref_collective  # noqa: E402
from wagma import optim as ref_optim  # noqa: E402
from wagma.netsim import MESSAGE, DelayModel, Simulator, StragglerPolicy  # noqa: E402
from wagma.problems import make_logistic, make_quadratic  # noqa: E402
from wagma.topology import (  # noqa: E402
    GroupingParams,
    InvalidParamsError,
    compute_groups,
    mixing_reachable,
    peer,
    phase_masks,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def groups_key(groups) -> str:
    return ";".join(",".join(str(r) for r in g) for g in groups)


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


# ---------------------------------------------------------------------------
# topology
# ---------------------------------------------------------------------------

def make_topology() -> dict:
    out = {"masks": {}, "groups_sha": {}, "groups_full": {}, "mixing": [], "peer": [],
           "invalid_params": [], "victims": []}
    P = 1
    while P <= 1024:
        log_p = int(math.log2(P))
        S = 1
        while S <= P:
            ts = list(range(max(1, 4 * log_p))) + [97, 1000, 12345]
            for t in ts:
                for rule in ("example", "literal"):
                    params = GroupingParams(P, S, t)
                    masks = phase_masks(params, rule).masks
                    key = f"{P},{S},{t},{rule}"
                    out["masks"][key] = list(masks)
                    part = compute_groups(params, rule)
                    gk = groups_key(part.groups)
                    out["groups_sha"][key] = sha(gk)
                    if P <= 32:
                        out["groups_full"][key] = [list(g) for g in part.groups]
            S *= 2
        P *= 2
    for P, S in [(2, 2), (8, 2), (8, 4), (8, 8), (16, 2), (16, 4), (32, 8), (64, 4), (64, 8)]:
        for rule in ("example", "literal"):
            for start in range(5):
                for k in range(1, int(math.log2(P)) + 2):
                    out["mixing"].append([P, S, start, k, rule,
                                          bool(mixing_reachable(GroupingParams(P, S, 0), start, k, rule))])
    for rank, mask, P in [(5, 4, 8), (0, 1, 8), (7, 2, 8), (8, 1, 8), (0, 3, 8), (0, 8, 8), (-1, 1, 8),
                          (1023, 512, 1024), (3, 0, 8)]:
        try:
            out["peer"].append([rank, mask, P, peer(rank, mask, P)])
        except InvalidParamsError:
            out["peer"].append([rank, mask, P, None])
    for P, S, t in [(3, 2, 0), (8, 3, 0), (4, 8, 0), (0, 1, 0), (8, 4, -1), (6, 1, 0), (8, 0, 0)]:
        try:
            GroupingParams(P, S, t)
            ok = True
        except InvalidParamsError:
            ok = False
        out["invalid_params"].append([P, S, t, ok])
    # straggler victim sets (netsim.py:75-82) -- numpy PCG64 draws
    for seed in (0, 2, 12, 99):
        for P in (4, 8, 16, 64):
            for k in (1, 2, 3):
                pol = StragglerPolicy(victims_per_iteration=k, extra_delay_ms=1.0, selection_seed=seed)
                for t in range(12):
                    out["victims"].append([seed, P, k, t, sorted(pol.victims(t, P))])
    return out


# ---------------------------------------------------------------------------
# collective (group round via the reference endpoints)
# ---------------------------------------------------------------------------

class _Node:
    def __init__(self, sim, rank, P, S, init, **kw):
        self.results = {}
        self.group = ref_collective.GroupAllreduce(sim, rank, P, S, on_complete=self._done,
                                                   initial_model=init, **kw)
        sim.register(rank, self._ev)

    def _done(self, version, acc, timely, stamp):
        self.results[version] = (acc.copy(), timely, stamp)

    def _ev(self, ev):
        if ev.kind == MESSAGE:
            src, body, _ = ev.payload
            self.group.handle_message(src, body)
        elif callable(ev.payload):
            ev.payload()


class _SyncNode:
    def __init__(self, sim, rank, P):
        self.results = {}
        self.sync = ref_collective.SyncAllreduce(sim, rank, P, on_complete=self._done)
        sim.register(rank, self._ev)

    def _done(self, it, total):
        self.results[it] = total.copy()

    def _ev(self, ev):
        if ev.kind == MESSAGE:
            src, body, _ = ev.payload
            self.sync.handle_message(src, body)
        elif callable(ev.payload):
            ev.payload()


def make_collective() -> dict:
    rng = np.random.default_rng(20050124)
    arrays: dict[str, np.ndarray] = {}
    cases = []
    d = 37
    idx = 0
    # (a) all timely group rounds: every rank joins at sim time 0
    for P in (2, 4, 8, 16):
        for S in (1, 2, 4, 8):
            if S > P:
                continue
            for rule in ("example", "literal"):
                for version in (0, 1, 2, 5):
                    sim = Simulator(P, link_latency_ms=1.0)
                    vecs = rng.standard_normal((P, d))
                    init = np.zeros((P, d))
                    nodes = [_Node(sim, r, P, S, init[r], mask_rule=rule) for r in range(P)]
                    for r in range(P):
                        nodes[r].group.join_or_check(version, vecs[r])
                    sim.run_until_idle()
                    acc = np.stack([nodes[r].results[version][0] for r in range(P)])
                    stamps = np.array([nodes[r].results[version][2] for r in range(P)], dtype=np.int64)
                    timely = np.array([nodes[r].results[version][1] for r in range(P)], dtype=np.int8)
                    arrays[f"c{idx}_fresh"] = vecs
                    arrays[f"c{idx}_stale"] = init
                    arrays[f"c{idx}_acc"] = acc
                    arrays[f"c{idx}_stamps"] = stamps
                    arrays[f"c{idx}_timely"] = timely
                    cases.append({"id": idx, "kind": "timely", "P": P, "S": S, "rule": rule,
                                  "version": version})
                    idx += 1
    # (b) stale participation: a subset of ranks joins much later; their
    #     stale send buffers (stamp -1) are pulled by the early activator
    for P, S in [(4, 2), (8, 2), (8, 4), (8, 8), (16, 4)]:
        for trial in range(4):
            sim = Simulator(P, link_latency_ms=1.0)
            stale = rng.standard_normal((P, d))
            fresh = rng.standard_normal((P, d))
            late = sorted(int(r) for r in rng.choice(P, size=max(1, P // 4), replace=False))
            nodes = [_Node(sim, r, P, S, stale[r]) for r in range(P)]
            for r in range(P):
                when = 1000.0 if r in late else float(rng.uniform(0.0, 0.2))
                sim.call_at(when, r, (lambda rr=r: nodes[rr].group.join_or_check(0, fresh[rr])))
            late_res = {}
            # rerun is not needed: ALREADY_DONE results are returned by the late joins
            orig = [n.group.join_or_check for n in nodes]
            for r in late:
                def wrap(version, vec, _r=r, _o=orig[r]):
                    res = _o(version, vec)
                    late_res[_r] = (res.status.value, None if res.accumulator is None else res.accumulator.copy())
                    return res
                nodes[r].group.join_or_check = wrap
            sim.run_until_idle()
            acc = np.stack([nodes[r].results[0][0] for r in range(P)])
            stamps = np.array([nodes[r].results[0][2] for r in range(P)], dtype=np.int64)
            timely = np.array([nodes[r].results[0][1] for r in range(P)], dtype=np.int8)
            arrays[f"c{idx}_fresh"] = fresh
            arrays[f"c{idx}_stale"] = stale
            arrays[f"c{idx}_acc"] = acc
            arrays[f"c{idx}_stamps"] = stamps
            arrays[f"c{idx}_timely"] = timely
            cases.append({"id": idx, "kind": "stale", "P": P, "S": S, "rule": "example", "version": 0,
                          "late": late, "late_status": {str(k): v[0] for k, v in late_res.items()}})
            idx += 1
    # (c) sync allreduce sums (collective.py:348-447)
    for P in (1, 2, 4, 8, 16):
        sim = Simulator(P, link_latency_ms=0.5)
        vecs = rng.standard_normal((P, d))
        nodes = [_SyncNode(sim, r, P) for r in range(P)]
        for r in range(P):
            sim.call_at(float(rng.uniform(0, 3)), r, (lambda rr=r: nodes[rr].sync.join(3, vecs[rr])))
        sim.run_until_idle()
        arrays[f"c{idx}_fresh"] = vecs
        arrays[f"c{idx}_acc"] = np.stack([nodes[r].results[3] for r in range(P)])
        cases.append({"id": idx, "kind": "sync", "P": P, "S": P, "rule": "example", "version": 3})
        idx += 1
    return {"arrays": arrays, "cases": cases}


# ---------------------------------------------------------------------------
# training trajectories
# ---------------------------------------------------------------------------

class _FixedVictims(StragglerPolicy):
    """Always slows rank 1 (mirrors `tests/test_optim.py:193-197`)."""

    def victims(self, iteration, P):
        return frozenset({1})


def record_training(name: str, P: int, opt, problem, delay, seed: int, mask_rule: str = "example"):
    grads: dict[tuple[int, int], np.ndarray] = {}
    etas: dict[tuple[int, int], float] = {}
    log: list[tuple[int, int, int]] = []
    orig_local_step = ref_optim.local_step
    orig_append = ref_optim._ContributionSink.append

    def rec_local_step(state, prob, partition, cfg, seed_, P_):
        from wagma.problems import draw_batch
        idx = draw_batch(partition, cfg.b, seed_, state.rank, state.iter)
        grads[(state.rank, state.iter)] = prob.batch_gradient(state.W, idx)
        etas[(state.rank, state.iter)] = cfg.eta.rate(state.iter, P_, cfg.T)
        return orig_local_step(state, prob, partition, cfg, seed_, P_)

    def rec_append(self, item):
        log.append(tuple(int(x) for x in item))
        return orig_append(self, item)

    ref_optim.local_step = rec_local_step
    ref_optim._ContributionSink.append = rec_append
    try:
        res = ref_optim.run_training(P, "wagma", opt, problem, delay, seed=seed, mask_rule=mask_rule)
    finally:
        ref_optim.local_step = orig_local_step
        ref_optim._ContributionSink.append = orig_append

    T, d = opt.T, problem.d
    G = np.zeros((T, P, d))
    E = np.zeros((T, P))
    for (r, t), g in grads.items():
        G[t, r] = g
        E[t, r] = etas[(r, t)]
    # contribution stamps per version; -2 = no group round at that version
    stamps = np.full((T, P), -2, dtype=np.int64)
    for r, v, s in log:
        assert stamps[v, r] == -2, "exactly-once violated in the reference?"
        stamps[v, r] = s
    meta = {"name": name, "P": P, "S": opt.S, "tau": opt.tau, "T": opt.T, "alpha": opt.alpha,
            "beta": opt.beta, "update_rule": opt.update_rule, "momentum": opt.momentum,
            "mask_rule": mask_rule, "max_staleness": res.max_staleness, "d": d,
            "sync_ok": [bool(ok) for _, ok in res.sync_replica_checks]}
    np.savez_compressed(os.path.join(HERE, f"training_{name}.npz"),
                        w0=problem.initial_point().astype(np.float64),
                        grads=G, etas=E, stamps=stamps,
                        final=np.stack(res.final_weights),
                        meta=np.array(json.dumps(meta)))
    if name in METRICS_CASES:
        recs = res.records
        prob = {"kind": problem.spec["kind"]}
        if prob["kind"] == "quadratic":
            arrays = {"eigs": problem.eigs, "x_star": problem.x_star}
        else:
            arrays = {"X": problem.X, "y": problem.y, "l2": np.array(problem.l2)}
        np.savez_compressed(os.path.join(HERE, f"metrics_{name}.npz"),
                            iteration=np.array([r.iteration for r in recs], dtype=np.int64),
                            loss_mu=np.array([r.loss_mu for r in recs]),
                            grad_norm_sq_mu=np.array([r.grad_norm_sq_mu for r in recs]),
                            gamma=np.array([r.gamma for r in recs]),
                            max_staleness=np.array([r.max_staleness for r in recs], dtype=np.int64),
                            csv=np.array(ref_optim.CSV_HEADER + "\n" + "\n".join(r.csv_row() for r in recs)),
                            problem=np.array(json.dumps(prob)), **arrays)
    return meta


# trajectories whose metrics rows are pinned (tests/test_gpu_metrics.py)
METRICS_CASES = ("logistic_p8s4_straggle", "quad_momentum_p8s2", "quad_s8_tau8")


def make_training():
    metas = []
    EtaS, Opt = ref_optim.EtaSchedule, ref_optim.OptimizerConfig
    logi = make_logistic(4096, 20, 1.0, seed=7)
    # config 1 (BASELINE.json configs[0]) shortened: no stragglers
    metas.append(record_training(
        "logistic_p8s4", 8, Opt(T=40, S=4, tau=10, alpha=True, eta=EtaS(value=0.5), b=16),
        logi, DelayModel(1.0, 0.0, 0.1), seed=5))
    # config 1 with the paper's straggler policy (2 victims, ~3.2x base delay)
    metas.append(record_training(
        "logistic_p8s4_straggle", 8, Opt(T=40, S=4, tau=10, alpha=True, eta=EtaS(value=0.5), b=16),
        logi, DelayModel(1.0, 0.3, 0.1, straggler=StragglerPolicy(2, 3.2, selection_seed=12)), seed=5))
    quad = make_quadratic(32, 5.0, seed=51)
    metas.append(record_training(
        "quad_momentum_p8s2", 8,
        Opt(T=24, S=2, tau=4, alpha=True, eta=EtaS(value=0.02), b=2, update_rule="momentum", momentum=0.9),
        quad, DelayModel(20.0, 5.0, 1.0, straggler=StragglerPolicy(3, 300.0, selection_seed=4)), seed=61))
    metas.append(record_training(
        "quad_s8_tau8", 8,
        Opt(T=32, S=8, tau=8, alpha=True, eta=EtaS(value=0.01), b=2, update_rule="momentum", momentum=0.9),
        quad, DelayModel(10.0, 2.0, 0.5, straggler=StragglerPolicy(2, 32.0, selection_seed=8)), seed=62))
    # S+1 rule (tests/test_optim.py:215-253)
    q8 = make_quadratic(8, 2.0, seed=7)
    metas.append(record_training(
        "fixed_victim_p4s2", 4, Opt(T=2, S=2, tau=None, alpha=True, eta=EtaS(value=0.05), b=1),
        q8, DelayModel(10.0, 0.0, 1.0, straggler=_FixedVictims(1, 5.0)), seed=33))
    # blocking group allreduce (beta)
    metas.append(record_training(
        "blocking_p4s4", 4, Opt(T=6, S=4, tau=None, alpha=False, beta=True, eta=EtaS(value=0.05), b=1),
        make_quadratic(8, 2.0, seed=6), DelayModel(10.0, 0.0, 1.0), seed=29))
    # literal mask rule with stragglers
    metas.append(record_training(
        "literal_p8s4", 8, Opt(T=20, S=4, tau=5, alpha=True, eta=EtaS(value=0.02), b=2),
        quad, DelayModel(10.0, 3.0, 1.0, straggler=StragglerPolicy(2, 40.0, selection_seed=3)), seed=9,
        mask_rule="literal"))
    # tau=1: every iteration is a global sync
    metas.append(record_training(
        "tau1_p4s2", 4, Opt(T=3, S=2, tau=1, alpha=True, eta=EtaS(value=0.1), b=2),
        make_quadratic(8, 2.0, seed=5), DelayModel(10.0, 0.0, 1.0), seed=13))
    # flags off: local SGD with sync every tau
    metas.append(record_training(
        "flags_off_p4", 4, Opt(T=7, S=2, tau=3, alpha=False, beta=False, eta=EtaS(value=0.07), b=2),
        make_quadratic(8, 2.0, seed=4), DelayModel(10.0, 0.0, 1.0), seed=17))
    # step eta schedule, P=16 S=4 with stragglers
    metas.append(record_training(
        "step_eta_p16s4", 16,
        Opt(T=30, S=4, tau=10, alpha=True, eta=EtaS(kind="step", value=0.05, decay_factor=0.5, decay_every=7), b=2),
        quad, DelayModel(5.0, 1.0, 0.2, straggler=StragglerPolicy(3, 16.0, selection_seed=21)), seed=44))
    return metas


def make_activation() -> list:
    """Counters after one version whose only activator is `root`: the root
    joins at t=0, every other rank long after the ACT tree and the phases ran."""
    out = []
    for P in (2, 4, 8, 16):
        for S in (2, 4):
            if S > P:
                continue
            for root in range(P):
                sim = Simulator(P, link_latency_ms=1.0)
                nodes = [_Node(sim, r, P, S, np.zeros(3)) for r in range(P)]
                for r in range(P):
                    when = 0.0 if r == root else 1000.0
                    sim.call_at(when, r, (lambda rr=r: nodes[rr].group.join_or_check(0, np.ones(3) * rr)))
                sim.run_until_idle()
                out.append({"P": P, "S": S, "root": root,
                            "acts_sent": [n.group.acts_sent for n in nodes],
                            "activations_originated": [n.group.activations_originated for n in nodes],
                            "phases_sent": [n.group.phases_sent for n in nodes]})
    return out


def main():
    act = make_activation()
    with open(os.path.join(HERE, "activation.json"), "w") as fp:
        json.dump(act, fp, separators=(",", ":"))
    if sys.argv[1:] == ["activation"]:
        return
    topo = make_topology()
    with open(os.path.join(HERE, "topology.json"), "w") as fp:
        json.dump(topo, fp, separators=(",", ":"))
    coll = make_collective()
    np.savez_compressed(os.path.join(HERE, "collective.npz"), **coll["arrays"],
                        cases=np.array(json.dumps(coll["cases"])))
    metas = make_training()
    for m in metas:
        print(m["name"], "max_staleness", m["max_staleness"])
    print("topology entries", len(topo["masks"]), "collective cases", len(coll["cases"]))


if __name__ == "__main__":
    main()
