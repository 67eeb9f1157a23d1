"""bench.py's contract on CPU: the workloads BASELINE.json names, and the
reference arm's JSON line (the oracle port on the host) with every key the
driver reads."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_workloads_cover_the_baseline_configs():
    sys.path.insert(0, str(ROOT))
    import bench

    shapes = {1: (2000, 1000, 8), 2: (20000, 5000, 8), 3: (200000, 20000, 8),
              4: (1000000, 40000, 4), 5: (500000, 20000, 8)}
    for c, (m, n, es) in shapes.items():
        W = bench.workload(c)
        assert (W["m"], W["n"], W["esize"]) == (m, n, es), c
        assert W["kind"] in ("fsvd", "rank")
    assert bench.workload(2)["kind"] == "rank" and bench.workload(2)["eps"] == 1e-6
    assert bench.workload(1)["k"] == 30 and bench.workload(1)["r"] == 10


@pytest.mark.timeout(600)
def test_reference_arm_line():
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=500)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert "workload" in line["config"]


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_bench_stdout_is_one_json_line_with_nccl():
    """Our arm through the multi-rank code path (NCCL initialised, which prints
    its version banner to fd 1 on some boxes): stdout must still be exactly
    the one JSON line the driver parses, with every key it reads."""
    import os

    env = {**os.environ, "KSVD_FORCE_NCCL": "1", "NCCL_DEBUG": "VERSION"}
    res = subprocess.run([sys.executable, "bench.py", "--config", "1", "--steps", "1",
                          "--warmup", "1", "--no-cpu-baseline"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=800)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = res.stdout.strip().splitlines()
    assert len(lines) == 1, res.stdout[:2000]
    line = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks", "stages_ms"):
        assert key in line, key
    assert line["value"] > 0 and line["gpu_launches"] > 0
    st = line["stages_ms"]
    assert st["gk_loop"] > 0 and st["spectral"] >= 0 and st["ritz_u_recovery_and_download"] > 0
