"""bench.py's reference arm on CPU: one JSON line with the driver's contract keys.

The reference arm times the oracle's C restatement of the reference arithmetic
(SURVEY.md §8(d)); it needs no GPU, so the line format is checked here.
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3",
                          "--nparams", "200000"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["steps"] == 3 and line["warmup"] == 3
    assert line["unit"] == "iters/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["config"]["workload"] and line["config"]["params_per_replica"] == 200000
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "iters/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_algorithmic_bytes_per_launch(monkeypatch):
    """Roofline numerators: pull leaves, split sums, hierarchical partials, one GPU."""
    import types

    b = _bench_module()
    n = 25_559_081
    N = 4.0 * n  # bytes per fp32 replica
    a = types.SimpleNamespace(P=8, S=8, tau=10, n=n)
    hbm, nvl = b.step_bytes(a, 1, 0, 0, 4)  # all 8 ranks local: 6 streams each, no NVLink
    assert nvl == 0 and hbm == 8 * 6 * N
    # hierarchical (opt-in, WG_HIER=1): 2 GPUs, masks (1,2,4): one 4-leaf partial per GPU, pull the other
    monkeypatch.setenv("WG_HIER", "1")
    hbm, nvl = b.step_bytes(a, 2, 0, 0, 4)
    assert nvl == 1.0 * N and hbm == 4 * 6 * N + N + N
    hbm, nvl = b.step_bytes(a, 4, 0, 0, 4)  # 4 GPUs: 2-leaf partials, reduce-scattered: 1/4*3 + 3/4
    assert nvl == 1.5 * N and hbm == 2 * 6 * N + N + 0.25 * N + 1.5 * N
    monkeypatch.setenv("WG_SPLIT", "0")
    hbm, nvl = b.step_bytes(a, 4, 0, 0, 4)  # without the split: pull the 3 other partials
    assert nvl == 3.0 * N and hbm == 2 * 6 * N + N + 3 * N
    monkeypatch.delenv("WG_SPLIT")
    assert b.hier_levels([0, 1, 2, 3, 4, 5, 6, 7], 4) == 2 and b.hier_levels([0, 4, 1, 5], 4) == 0
    assert b.hier_levels([0, 2, 4, 6], 4) == 1 and b.hier_levels([0, 1, 2, 3], 4) == 0  # one GPU: no exchange
    monkeypatch.setenv("WG_HIER", "0")
    hbm, nvl = b.step_bytes(a, 4, 0, 0, 4)  # split over 4 GPUs: f = 2/8 -> f*6 + 3/4 = 2.25 N
    assert nvl == 2.25 * N and hbm == 2 * 6 * N + 0.25 * N + 2.25 * N
    hbm, nvl = b.step_bytes(a, 8, 0, 0, 4)  # one rank per GPU: 1/8*7 + 7/8 = 1.75 N
    assert nvl == 1.75 * N
    a = types.SimpleNamespace(P=4, S=2, tau=10, n=n)
    hbm, nvl = b.step_bytes(a, 4, 0, 0, 4)  # S=2 pairs across GPUs: split does not pay, pull 1 leaf
    assert nvl == N and hbm == 6 * N + N
    a = types.SimpleNamespace(P=4, S=4, tau=10, n=262_144)  # 1 MiB: below the split threshold
    hbm, nvl = b.step_bytes(a, 4, 0, 0, 4)
    assert nvl == 3 * 4.0 * 262_144


def test_large_replicas_sum_leaves_at_four_gpus(monkeypatch):
    """Above WG_HIER_SPLIT_MAX_BYTES (160 MiB) a launch whose partials would be
    reduce-scattered sums leaves instead (wg_launch); 2 GPUs keep the partials."""
    import types

    b = _bench_module()
    n = 213_000_000
    N = 4.0 * n
    a = types.SimpleNamespace(P=8, S=8, tau=8, n=n)
    monkeypatch.delenv("WG_HIER", raising=False)
    hbm, nvl = b.step_bytes(a, 4, 0, 0, 4)  # leaf-level split: 2.25 N
    assert nvl == 2.25 * N
    hbm, nvl = b.step_bytes(a, 2, 0, 0, 4)  # 2 GPUs: pull the other GPU's partial
    assert nvl == 1.0 * N
    monkeypatch.setenv("WG_HIER_SPLIT_MAX_BYTES", str(1 << 40))
    hbm, nvl = b.step_bytes(a, 4, 0, 0, 4)
    assert nvl == 1.5 * N
