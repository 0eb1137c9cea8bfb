"""bench.py's reference arm (the oracle port timed on the host):
runs on CPU, prints one JSON line with the contract's keys, and states the
host threads it used."""

import json
import os
import subprocess
import sys

from conftest import REPO


def test_reference_arm_json_line():
    env = dict(os.environ, PYTHONPATH=REPO)
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
         "--config", "c2", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines            # stdout carries the JSON line only
    line = json.loads(lines[0])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
                "ms_per_step", "higher_is_better", "config", "e2e",
                "cpu_baseline"):
        assert key in line
    assert line["value"] > 0 and line["unit"] == "charges/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == line["value"]
    assert cb["cores"] == len(os.sched_getaffinity(0))
    # the same config dict as the GPU arm (bench.bench_config), so the
    # driver can match the two lines
    sys.path.insert(0, REPO)
    import bench
    from paper_2101_07088_b200 import workloads as W
    system, params = W.build("c2")

    class A:
        config, replicate_grid = "c2", False
    assert line["config"] == json.loads(json.dumps(bench.bench_config(A, system, params)))
    assert line["extrapolated"] is True and line["sample_wall_s"]["total"] > 0


def test_cpu_bench_workers_match_single_thread_grid():
    """The FFT workers knob changes the timing only: the oracle grid stages
    run with workers > 1 (the reference's threads parameter)."""
    from oracle import cpu_bench
    from paper_2101_07088_b200 import workloads as W
    system, params = W.build("c1")
    t1 = cpu_bench.grid_stage_seconds(system, params, workers=1)
    t2 = cpu_bench.grid_stage_seconds(system, params, workers=2)
    assert t1 > 0 and t2 > 0
