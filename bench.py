"""WAGMA group-averaging benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W

Workload (BASELINE.json configs[1]): ResNet-50-sized replicas, N = 25,559,081
fp32 parameters, P = 8 WAGMA ranks, group size S = 8 (north-star target),
tau = 10, momentum SGD (eta 0.1, beta 0.9), wait-avoiding activation. The P
ranks are mapped block-wise onto the N GPUs (rank r on GPU r // (P/N)), so
total work is fixed as N grows ("scaling": "strong"). A step is one WAGMA
iteration of all P ranks = one fused kernel launch per GPU (local momentum
step + send-ring install + group / global average). Synthetic data: W0 ~
N(0, 0.02^2) identical on every rank, g ~ N(0, 0.01^2) (two pre-generated
gradient buffers per rank, alternated), inputs resident in HBM.

`--impl reference` times the reference path's CPU implementation on the host
cores: the C restatement of the reference arithmetic in oracle/ (the
reference itself is Python and does not exist on the GPU box), on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "WAGMA iters/s and group-avg GB/s vs NVLink roofline at 1/2/4/8 B200"
N_RESNET50 = 25_559_081
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
NVLINK_NOMINAL_GBS = 900.0  # nominal per direction per GPU (north_star)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "nccl"])
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--S", type=int, default=8)
    ap.add_argument("--nparams", type=int, default=N_RESNET50, dest="n")
    ap.add_argument("--tau", type=int, default=10)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps (capped at 60)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--grace-us", type=float, default=100.0)
    # imbalance experiments (not part of the default metric line)
    ap.add_argument("--blocking", action="store_true", help="blocking group allreduce (beta) instead of alpha")
    ap.add_argument("--base-ms", type=float, default=0.0, help="device-side 'compute' delay per step, every GPU")
    ap.add_argument("--victims", type=int, default=0, help="StragglerPolicy victims per iteration")
    ap.add_argument("--extra-ms", type=float, default=0.0, help="extra delay of a victim rank's GPU")
    ap.add_argument("--straggler-seed", type=int, default=12)
    ap.add_argument("--fixed-victim", type=int, default=-1,
                    help="C4: this rank is the victim of every iteration (_FixedVictims, tests/test_optim.py:193-197)")
    ap.add_argument("--length-buckets", action="store_true",
                    help="C3: per-(rank, t) compute time base_ms * L / mean(L), L from WMT-style length buckets")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fp:
            d = json.load(fp)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def workload_name(a):
    model = "ResNet-50-sized" if a.n == N_RESNET50 else f"n={a.n}"
    return f"{model} WAGMA group averaging, P={a.P} ranks, S={a.S}, tau={a.tau}, momentum"


def config_dict(a, G):
    return {"workload": workload_name(a), "params_per_replica": a.n, "ranks": a.P, "group_size": a.S,
            "tau": a.tau, "update_rule": "momentum", "eta": 0.1, "beta": 0.9, "activation": "wait-avoiding",
            "rank_mapping": f"block ({a.P // G} ranks per GPU)", "parallelism": f"wagma-p{a.P}-g{G}",
            "l2": "inputs larger than L2 (every step streams all replicas, > 1 GB)"}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle's C restatement of the reference arithmetic
# ---------------------------------------------------------------------------

def cpu_port_run(a, steps: int, warmup: int, seconds: float):
    """Time the C port (OpenMP, all host threads) on the same workload.

    Returns (iters_per_s, threads, sample_description, per_iter_s)."""
    from oracle import c_oracle
    from oracle import topology_oracle as otopo
    dt = np.float32 if a.dtype == "f32" else np.float64
    P, n = a.P, a.n
    rng = np.random.default_rng(1234)
    w0 = (rng.standard_normal(n) * 0.02).astype(dt)
    W = [w0.copy() for _ in range(P)]
    m = [np.zeros(n, dt) for _ in range(P)]
    g = [(rng.standard_normal(n) * 0.01).astype(dt) for _ in range(P)]
    wp = [np.empty(n, dt) for _ in range(P)]
    threads = c_oracle.max_threads()

    def one(t):
        sync = (t + 1) % a.tau == 0
        masks = [1 << j for j in range(P.bit_length() - 1)] if sync else list(otopo.phase_masks(P, a.S, t))
        c_oracle.wagma_iteration(W, m, g, wp, masks, P if sync else a.S, 0.1, 0.9, True, nthreads=threads)

    for t in range(warmup):
        one(t)
    times = []
    t0 = time.perf_counter()
    t = warmup
    while len(times) < steps:
        s = time.perf_counter()
        one(t)
        times.append(time.perf_counter() - s)
        t += 1
        if seconds and time.perf_counter() - t0 > seconds and len(times) >= 2:
            break
    total = sum(times)
    sample = (f"{len(times)} iterations of P={P} ranks x N={n} {a.dtype} (local step + S={a.S} group sums "
              f"in the reference's recursive-doubling order + averaging), C/OpenMP port of the reference "
              f"arithmetic, {threads} threads")
    return len(times) / total, threads, sample, total / len(times)


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ips, threads, sample, _ = cpu_port_run(a, a.steps, a.warmup, seconds=a.cpu_seconds * 3)
    line = {"metric": METRIC, "value": ips, "unit": "iters/s", "impl": "reference", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000.0 / ips, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
            "config": config_dict(a, max(1, a.gpus)),
            "cpu_baseline": {"value": ips, "unit": "iters/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": ips, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as fp:
            for line in fp:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# algorithmic bytes
# ---------------------------------------------------------------------------

def hier_levels(leaves, R):
    """Tree levels of a plan summed inside one GPU (the kernel's plan_hl, 0 = none).

    Largest h >= 1 such that every block of 2^h consecutive leaves lives on
    one GPU under the block mapping, for plans that span >= 2 GPUs with
    distinct leaves (mirrors wg_launch)."""
    n = len(leaves)
    if len({q // R for q in leaves}) < 2 or len(set(leaves)) != n:
        return 0
    log = n.bit_length() - 1
    for h in range(log - 1, 0, -1):
        if all(leaves[i] // R == leaves[i & ~((1 << h) - 1)] // R for i in range(n)):
            return h
    return 0


def step_bytes(a, G, gpu_index, t, elem):
    """(HBM bytes, NVLink ingress bytes) one launch on `gpu_index` must move.

    Own streams per local rank: read W, m, g; write m, the send-slot W' and
    W_{t+1} = 6 * elem * n. Bytes read from this GPU by peers (symmetric)
    are added to its HBM. The kernel's own re-reads of data it just wrote
    (local leaves or partials copied into shared memory) are not counted
    (SURVEY.md §8(d)). Per plan, the algorithm the kernel runs:
    - hierarchical (all timely, lowest hl tree levels inside one GPU,
      WG_HIER): each GPU writes its 2^hl-leaf subtree partials once and pulls
      the other GPUs' partials: NVLink = remote partials, HBM += local partials;
    - split (all timely, spans >= 2 GPUs where it saves bytes, P <= 8, the
      kernel's split_pays; only when no plan of the launch is hierarchical):
      a fraction f = L/S of the tiles is reduced here (S - L remote leaves
      each, the reduced tile written), the rest arrive as one reduced tile;
    - pull: every leaf on another GPU crosses NVLink once.
    """
    from paper_2005_00124_b200.topology import GroupingParams, compute_groups, tree_leaves
    R = a.P // G
    local = range(gpu_index * R, (gpu_index + 1) * R)
    n = elem * a.n
    hbm = R * 6 * n
    nvl = 0.0
    sync = (t + 1) % a.tau == 0
    groups = [tuple(range(a.P))] if sync else None
    if not sync:
        part = compute_groups(GroupingParams(a.P, a.S, t))
        groups = []
        for r in local:
            grp = part.group_of(r)
            if grp not in groups:
                groups.append(grp)
    plans = [(grp, list(grp) if sync else list(tree_leaves(GroupingParams(a.P, a.S, t), grp[0]))) for grp in groups]
    hier_on = os.environ.get("WG_HIER", "1") != "0" and G >= 2
    hls = [hier_levels(leaves, R) if hier_on else 0 for _, leaves in plans]
    split_on_h = os.environ.get("WG_SPLIT", "1") != "0" and G >= 2 and a.P <= 8 and \
        n >= int(os.environ.get("WG_SPLIT_MIN_BYTES", str(8 << 20)))  # the kernel's split_min_bytes
    # the kernel sums leaves when its partials would be reduce-scattered and the
    # replica exceeds WG_HIER_SPLIT_MAX_BYTES (mirrors wg_launch)
    span_min = int(os.environ.get("WG_SPLIT_SPAN", "2"))

    def pays(leaves, hl):
        parts = leaves[::1 << hl]
        sp = len({q // R for q in parts})
        return sp >= span_min and 2 * len(parts) >= 3 * (len(parts) // sp + 1)
    wide_h = any(hl and pays(leaves, hl) for (_, leaves), hl in zip(plans, hls))
    if wide_h and os.environ.get("WG_MG", "0") == "0" and \
            n > int(os.environ.get("WG_HIER_SPLIT_MAX_BYTES", str(160 << 20))):
        hls = [0] * len(hls)
    split_on = split_on_h and not any(hls)
    for (grp, leaves), hl in zip(plans, hls):
        L = sum(1 for q in grp if q // R == gpu_index)
        S = len(grp)
        spans = len({q // R for q in grp})
        if hl:
            parts = leaves[::1 << hl]
            ne = len(parts)
            local_parts = sum(1 for q in parts if q // R == gpu_index)
            hbm += n * local_parts  # this GPU's partials, written once
            pspans = len({q // R for q in parts})
            if split_on_h and pspans >= int(os.environ.get("WG_SPLIT_SPAN", "2")) and 2 * ne >= 3 * (ne // pspans + 1):
                # partials reduce-scattered over their keys: a fraction f of the
                # tiles is reduced here from the other GPUs' partials, the rest
                # arrive as one reduced tile (the reduced tiles written: f)
                f = local_parts / ne
                nvl += n * (f * (ne - local_parts) + (1 - f))
                hbm += n * f
            else:
                nvl += n * (ne - local_parts)
        elif split_on and spans >= int(os.environ.get("WG_SPLIT_SPAN", "2")) and 2 * S >= 3 * (S // spans + 1) and \
                len(set(leaves)) == len(leaves):
            f = L / S
            nvl += n * (f * (S - L) + (1 - f))
            hbm += n * f
        else:
            nvl += n * sum(1 for q in leaves if q // R != gpu_index)
    return hbm + nvl, nvl


def load_traffic(a, G):
    """dram bytes per launch from a committed ncu --set full capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as fp:
        d = json.load(fp)
    key = f"P{a.P}_S{a.S}_n{a.n}_{a.dtype}_g{G}"
    v = d.get(key)
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_2005_00124_b200.context import DeviceContext
    from paper_2005_00124_b200.dist import max_over_ranks
    from paper_2005_00124_b200.optim import EtaSchedule, GroupAveragingOptimizer, OptimizerConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    G = world
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    dt = torch.float32 if a.dtype == "f32" else torch.float64
    elem = 4 if a.dtype == "f32" else 8
    if a.P % G:
        raise SystemExit(f"P={a.P} must be divisible by the GPU count {G}")

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x: float) -> float:
        return max_over_ranks(x, device=dev)

    ctx = DeviceContext(a.P, a.S, a.n, dtype=dt, tau=a.tau, n_gpus=G, gpu_index=rank, device=dev.index,
                        grace_us=a.grace_us, timeout_s=30.0, activation_enabled=not a.blocking)
    cfg = OptimizerConfig(T=1 << 30, S=a.S, tau=a.tau, alpha=not a.blocking, beta=a.blocking,
                          eta=EtaSchedule(value=0.1), update_rule="momentum", momentum=0.9)
    from paper_2005_00124_b200.straggler import StragglerPolicy
    policy = StragglerPolicy(a.victims, a.extra_ms, selection_seed=a.straggler_seed) if a.victims else None
    if a.fixed_victim >= 0:
        from paper_2005_00124_b200.straggler import FixedVictims
        policy = FixedVictims(a.fixed_victim, a.extra_ms)

    from paper_2005_00124_b200.straggler import BucketedLengthDelay
    lengths = BucketedLengthDelay(a.base_ms, seed=a.straggler_seed) if a.length_buckets else None

    def delay(t):
        """compute_delay (netsim.py:103-117) as a device spin before this GPU's step."""
        ms = a.base_ms if lengths is None else max(lengths.delay_ms(r, t) for r in local)
        if policy is not None and set(local) & policy.victims(t, a.P):
            ms += a.extra_ms
        if ms > 0:
            ctx.delay(int(ms * 1e6))
    gen = torch.Generator(device=dev).manual_seed(1234)
    w0 = torch.randn(a.n, generator=gen, device=dev, dtype=dt) * 0.02
    opt = GroupAveragingOptimizer(ctx, cfg, w0)
    local = list(ctx.local_ranks)
    gpool = {r: [torch.randn(a.n, generator=gen, device=dev, dtype=dt) * 0.01 for _ in range(2)] for r in local}
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    barrier()

    t = 0
    for _ in range(a.warmup):
        delay(t)
        opt.step(t, {r: gpool[r][t % 2] for r in local})
        t += 1
    sampler = ClockSampler(dev.index) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    torch.cuda.synchronize()
    barrier()
    launches0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_first = t
    start.record(stream)
    for k in range(a.steps):
        delay(t)
        ev[k][0].record(stream)
        opt.step(t, {r: gpool[r][t % 2] for r in local})
        ev[k][1].record(stream)
        t += 1
    end.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    gpu_launches = ctx.launches - launches0
    ctx.check()
    # contribution stamps the activation protocol locked for the last timed
    # versions (descriptor ring): how many contributions were stale
    stale = total_c = 0
    from paper_2005_00124_b200.optim import is_sync_iteration
    for v in range(max(t_first, t - ctx.ring_depth + 1), t):
        if is_sync_iteration(v, a.tau) or a.blocking:
            continue
        stamps, locked = ctx.query_version(v)
        if locked:
            total_c += len(stamps)
            stale += sum(1 for st in stamps if st != v)
    protocol = {"stale_contributions": stale, "contributions": total_c}
    elapsed_ms = allmax(start.elapsed_time(end))
    kern_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(a.steps)]
    kern_avg_ms = allmax(sum(kern_ms) / len(kern_ms))
    ms_per_step = elapsed_ms / a.steps
    iters_per_s = 1000.0 * a.steps / elapsed_ms

    # algorithmic bytes of the dominant (only) kernel, averaged over the timed steps
    hbm_b, nvl_b = 0, 0
    for tt in range(t_first, t_first + a.steps):
        h, v = step_bytes(a, G, rank, tt, elem)
        hbm_b += h
        nvl_b += v
    hbm_b /= a.steps
    nvl_b /= a.steps
    hbm_peak, peak_kind = measured_peaks()
    t_hbm = hbm_b / (hbm_peak * 1e9)
    t_nvl = nvl_b / (NVLINK_PEER_GBS * 1e9)
    kern_s = kern_avg_ms / 1e3
    if t_nvl > t_hbm:
        roof = {"bound": "nvlink", "achieved": nvl_b / kern_s / 1e9, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 nominal)"}
    else:
        roof = {"bound": "hbm", "achieved": hbm_b / kern_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "peak_source": f"{peak_kind} HBM copy (MEASURED_PEAKS.json)"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    if nvl_b:
        roof["nvlink_frac"] = {"of_770_measured": nvl_b / kern_s / 1e9 / NVLINK_PEER_GBS,
                               "of_900_nominal": nvl_b / kern_s / 1e9 / NVLINK_NOMINAL_GBS}
    roof["t_star_frac"] = {"measured_peaks": max(t_hbm, t_nvl) / kern_s,
                           "nominal_900": max(t_hbm, nvl_b / (NVLINK_NOMINAL_GBS * 1e9)) / kern_s}
    roof["traffic"] = load_traffic(a, G)
    roof["traffic_source"] = (
        "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch)"
        if roof["traffic"] is not None else
        "none: ncu cannot wrap a multi-rank run and NVML NVLink/DRAM counters are not supported on this pool"
        if G > 1 else "none: no committed ncu capture for this config")
    roof["algorithmic_bytes_per_launch"] = {"hbm": hbm_b, "nvlink_ingress": nvl_b}
    roof["kernel_ms"] = kern_avg_ms
    roof["roofline_ms"] = max(t_hbm, t_nvl) * 1e3
    group_avg_gbs = nvl_b / kern_s / 1e9 if nvl_b else 0.0

    # end to end through the public API with host buffers: every step copies
    # its gradients in from pinned host memory and its averaged replicas back
    # out. Copies run on two side streams (PCIe is full duplex): step k's
    # gradients come in while step k-1's replicas (snapshotted on device right
    # after its step) go out; the step itself waits for its own inputs.
    e2e = None
    if not a.no_e2e:
        ke = a.e2e_steps or min(a.steps, 60)
        ghost = {r: [gp.cpu().pin_memory() for gp in gpool[r]] for r in local}
        whost = {r: [torch.empty(a.n, dtype=dt).pin_memory() for _ in range(2)] for r in local}
        gdev = {r: [torch.empty(a.n, dtype=dt, device=dev) for _ in range(2)] for r in local}
        wsnap = {r: [torch.empty(a.n, dtype=dt, device=dev) for _ in range(2)] for r in local}
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        in_done, step_done, out_done = [None] * ke, [None] * ke, [None] * ke
        torch.cuda.synchronize()
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        for k in range(ke):
            b = k % 2
            with torch.cuda.stream(s_in):
                if k >= 2:
                    s_in.wait_event(step_done[k - 2])  # gdev[b] free again
                for r in local:
                    gdev[r][b].copy_(ghost[r][t % 2], non_blocking=True)
                in_done[k] = ev()
                in_done[k].record(s_in)
            stream.wait_event(in_done[k])
            if k >= 2:
                stream.wait_event(out_done[k - 2])  # wsnap[b] drained
            opt.step(t, {r: gdev[r][b] for r in local})
            for r in local:
                wsnap[r][b].copy_(opt.W[r], non_blocking=True)
            step_done[k] = ev()
            step_done[k].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(step_done[k])
                for r in local:
                    whost[r][b].copy_(wsnap[r][b], non_blocking=True)
                out_done[k] = ev()
                out_done[k].record(s_out)
            t += 1
        stream.wait_event(out_done[ke - 1])
        s1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = allmax(s0.elapsed_time(s1))
        e2e = {"value": 1000.0 * ke / e2e_ms, "unit": "iters/s", "h2d_bytes_per_step": len(local) * elem * a.n,
               "d2h_bytes_per_step": len(local) * elem * a.n, "steps": ke,
               "path": "pinned host gradients -> GroupAveragingOptimizer.step -> pinned host replicas "
                       "(H2D and D2H on two copy streams, overlapped across steps)"}
        ctx.check()

    # sanity (untimed): replicas finite; run on to the next global sync and
    # check the replicas are bit-identical there (optim.py:289-293)
    for r in local:
        if not torch.isfinite(opt.W[r]).all():
            raise SystemExit(f"non-finite replica on rank {r}")
    from paper_2005_00124_b200.diagnostics import replica_diagnostics
    while (t + 1) % a.tau != 0:
        delay(t)
        opt.step(t, {r: gpool[r][t % 2] for r in local})
        t += 1
    delay(t)
    opt.step(t, {r: gpool[r][t % 2] for r in local})
    t += 1
    diag = replica_diagnostics(ctx, opt.W)
    ctx.check()

    cpu = None
    if rank == 0 and G == 1 and not a.no_cpu:
        ips, threads, sample, _ = cpu_port_run(a, 1000, 1, seconds=a.cpu_seconds)
        cpu = {"value": ips, "unit": "iters/s", "cores": threads, "kind": "port", "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": iters_per_s, "unit": "iters/s", "n_gpus": G, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": a.dtype, "data": "synthetic", "config": config_dict(a, G),
                "group_avg_gbs": group_avg_gbs, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": gpu_launches, "clocks": clocks, "protocol_last_versions": protocol,
                "replicas_after_sync": {"iteration": t - 1, "bit_identical": diag.identical, "gamma": diag.gamma}}
        if a.blocking or a.victims or a.base_ms or a.length_buckets or a.fixed_victim >= 0:
            from paper_2005_00124_b200.optim import is_sync_iteration
            stale = total = 0
            for v in range(max(0, t - ctx.ring_depth + 1), t):
                if is_sync_iteration(v, a.tau) or a.blocking:
                    continue
                stamps, locked = ctx.query_version(v)
                if locked:
                    total += len(stamps)
                    stale += sum(1 for st in stamps if st != v)
            line["imbalance"] = {"activation": "blocking (beta)" if a.blocking else "wait-avoiding (alpha)",
                                 "base_ms": a.base_ms, "victims_per_iteration": a.victims, "extra_ms": a.extra_ms,
                                 "fixed_victim": a.fixed_victim if a.fixed_victim >= 0 else None,
                                 "selection_seed": a.straggler_seed,
                                 "delay_model": "bucketed sequence lengths (WMT-style)" if a.length_buckets
                                 else "base + victims",
                                 "stale_contribution_fraction": (stale / total) if total else None}
            line["config"]["activation"] = line["imbalance"]["activation"]
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# NCCL sub-communicator baseline (comparison only; one WAGMA rank per GPU)
# ---------------------------------------------------------------------------

def run_nccl(a):
    """torch momentum step + ncclAllReduce(AVG) on per-group sub-communicators.

    Blocking (beta) semantics: every rank waits for its whole group. One rank
    per GPU (NCCL cannot host several ranks of a communicator on one GPU), so
    P = world size; groups come from the same schedule (compute_groups), one
    communicator per distinct group of the schedule period (ncclCommSplit via
    torch.distributed.new_group), the global sync every tau iterations.
    """
    import torch
    import torch.distributed as dist

    from paper_2005_00124_b200.dist import max_over_ranks
    from paper_2005_00124_b200.topology import GroupingParams, compute_groups

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    P, S = world, min(a.S, world)
    dt = torch.float32 if a.dtype == "f32" else torch.float64
    period = max(1, (P.bit_length() - 1)) if P > 1 else 1
    comms = {}
    for t in range(period):
        for grp in compute_groups(GroupingParams(P, S, t)).groups:
            if grp not in comms and len(grp) > 1:
                comms[grp] = dist.new_group(list(grp)) if world > 1 else None
    gen = torch.Generator(device=dev).manual_seed(1234)
    W = torch.randn(a.n, generator=gen, device=dev, dtype=dt) * 0.02
    m = torch.zeros_like(W)
    gpool = [torch.randn(a.n, generator=gen, device=dev, dtype=dt) * 0.01 for _ in range(2)]

    def step(t):
        m.mul_(0.9).add_(gpool[t % 2])
        W.sub_(m, alpha=0.1)
        if world == 1:
            return
        if (t + 1) % a.tau == 0:
            dist.all_reduce(W, op=dist.ReduceOp.AVG)
        else:
            grp = compute_groups(GroupingParams(P, S, t)).group_of(rank)
            if len(grp) > 1:
                dist.all_reduce(W, op=dist.ReduceOp.AVG, group=comms[grp])

    for t in range(a.warmup):
        step(t)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for t in range(a.warmup, a.warmup + a.steps):
        step(t)
    s1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(s0.elapsed_time(s1), device=dev) / a.steps
    if rank == 0:
        elem = 4 if a.dtype == "f32" else 8
        busbw = 2 * (S - 1) / S * elem * a.n / (ms / 1e3) / 1e9 if S > 1 else 0.0
        cfg = config_dict(a, world)
        cfg.update({"ranks": P, "group_size": S, "rank_mapping": "one rank per GPU",
                    "parallelism": f"nccl-subcomm-p{P}-g{world}", "activation": "blocking (beta)"})
        print(json.dumps({"metric": METRIC, "value": 1000.0 / ms, "unit": "iters/s", "impl": "nccl",
                          "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": a.dtype,
                          "data": "synthetic", "config": cfg, "nccl_busbw_gbs": busbw}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.impl == "nccl":
        run_nccl(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
