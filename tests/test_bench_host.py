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
