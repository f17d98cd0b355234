"""CPU: bench.py's CPU-baseline leg (the oracle port timed in both of SURVEY.md §8d's modes) —
structure of the reported block, no GPU needed."""

import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("cfg", ["1", "3"])
def test_cpu_baseline_reports_both_modes(cfg):
    b = _bench()
    r = b.cpu_baseline(cfg, budget_s=0.6)
    assert r["kind"] == "port" and r["cores"] >= 1 and r["value"] > 0
    modes = r["modes"]
    assert set(modes) == {"pool", "single"}
    best = min(modes, key=lambda m: modes[m]["step_seconds"])
    assert r["best_mode"] == best
    assert r["step_seconds"] == pytest.approx(modes[best]["step_seconds"])
    units = {"1": 65_536, "3": 1.0}[cfg]
    assert r["value"] == pytest.approx(units / r["step_seconds"], rel=1e-9)


def test_cpu_baseline_records_host_provenance():
    r = _bench().cpu_baseline("1", budget_s=0.3)
    host = r["host"]
    assert host["nproc"] >= 1 and host["numpy"]
    assert "cpu_model" in host and "blas" in host


def test_cpu_baseline_solve_both_modes():
    r = _bench().cpu_baseline("solve", budget_s=0.5)
    assert set(r["modes"]) == {"single", "single_1blas", "pool"} and r["cores"] >= 1
    assert r["best_mode"] in r["modes"]


def test_gpus_flag_fails_loudly_without_gpus():
    """bench.py --gpus 2 outside torchrun re-launches itself as 2 ranks, or exits non-zero with a
    message when fewer GPUs are visible (this container has none)."""
    import subprocess
    import sys

    import torch

    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        pytest.skip("has 2 GPUs: the relaunch would really run")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode != 0
    assert "--gpus 2 needs 2 visible CUDA devices" in p.stderr


def test_world_size_mismatch_is_an_error():
    import subprocess
    import sys

    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode == 2 and "WORLD_SIZE=3" in p.stderr
