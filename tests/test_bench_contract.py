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


def test_rank_envs():
    sys.path.insert(0, str(ROOT))
    import bench

    envs = bench.rank_envs(2, 12345, base={"PATH": "/bin"})
    assert [e["RANK"] for e in envs] == ["0", "1"]
    assert [e["LOCAL_RANK"] for e in envs] == ["0", "1"]
    assert all(e["WORLD_SIZE"] == "2" and e["MASTER_ADDR"] == "127.0.0.1"
               and e["MASTER_PORT"] == "12345" and e["NCCL_DEBUG"] == "INFO" for e in envs)
    one = bench.rank_envs(1, 1, base={})[0]
    assert one["WORLD_SIZE"] == "1" and "NCCL_DEBUG" not in one


@pytest.mark.timeout(300)
def test_launcher_env_plumbing(tmp_path):
    """bench.launch() at N=2 (what `bench.py --gpus 2` does) on CPU: both
    ranks rendezvous over gloo from the environment it sets."""
    code = ("import sys, bench; sys.exit(bench.launch(2, [sys.argv[1]], "
            "script='tests/launch_probe.py', check_gpus=False))")
    res = subprocess.run([sys.executable, "-c", code, str(tmp_path)], cwd=ROOT,
                         capture_output=True, text=True, timeout=280)
    assert res.returncode == 0, res.stderr[-2000:]
    recs = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(2)]
    assert [r["RANK"] for r in recs] == ["0", "1"]
    assert all(r["sum"] == 3.0 and r["WORLD_SIZE"] == "2" for r in recs)
    assert res.stdout.strip() == "rank0-stdout"


def test_launcher_refuses_missing_gpus():
    """More GPUs asked for than visible: non-zero exit, no JSON line."""
    res = subprocess.run([sys.executable, "bench.py", "--gpus", "64", "--config", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert res.returncode != 0 and res.stdout.strip() == ""
    assert "GPU(s) visible" in res.stderr


def test_world_size_mismatch_refused():
    env = {**__import__("os").environ, "WORLD_SIZE": "2", "RANK": "0"}
    res = subprocess.run([sys.executable, "bench.py", "--gpus", "1", "--config", "1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert res.returncode == 2 and "WORLD_SIZE" in res.stderr
