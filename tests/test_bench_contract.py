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
