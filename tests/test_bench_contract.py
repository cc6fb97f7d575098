"""bench.py's host-side contract, on CPU: the reference arm (`--impl reference`,
the unmodified reference from oracle/_ref on the host cores) prints one JSON line
with the keys the driver reads and the same `config` dict the GPU arm prints; the
seeded SFI schedule follows the reference's step rule (scheduler.cpp:93-99); the
C5 slow fractions fall as t_max grows."""
from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    import bench

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["metric"] == bench.metric_name("c1") and line["unit"] == "tokens/s" and line["value"] > 0
    assert line["warmup"] >= 3 and line["higher_is_better"] is True
    assert line["config"] == bench.config_dict("c1", 1)  # the GPU arm prints the same dict
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert cb["single_thread"]["value"] > 0
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_schedule_follows_the_step_rule():
    import bench

    sched = bench.schedule(2000, seed=7)
    assert sched[0]  # step 0 is slow (init_decode_state)
    since = 0
    for s in sched[1:]:
        since = 0 if s else since + 1
        assert since + 1 <= bench.T_MAX  # a slow step at the latest when steps_since_slow + 1 >= t_max
    frac = sum(sched) / len(sched)
    assert 1 / bench.T_MAX < frac < 0.1  # triggers p = 1/24 plus the forced refreshes


def test_c5_slow_fraction_decreases_with_t_max():
    import bench

    f = [bench.c5_slow_fraction(t, 32768) for t in bench.C5_TMAX]
    assert all(a > b for a, b in zip(f, f[1:]))
    assert all(1 / 24 < x < 0.1 for x in f)
