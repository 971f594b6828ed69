"""bench.py's reference arm runs on the host alone: its JSON line carries the
contract's keys (metric/value/unit, impl, cpu_baseline, e2e with no copies),
and under torchrun only rank 0 prints."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)


def test_reference_arm_line():
    p = _run(None, "--config", "lenet", "--steps", "2", "--warmup", "1")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    ref_present = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "weightpack"))
    assert d["cpu_baseline"]["kind"] == ("reference" if ref_present else "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("lenet")
    assert d["config"]["weights"] == 430500 and d["config"]["algorithmic_bytes_per_step"] == 2 * 5 * 430500


def test_reference_arm_config_matches_ours():
    """Both arms build `config` from the same function: the driver's same_config check."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    p = _run(None, "--config", "lenet", "--steps", "1", "--warmup", "0")
    d = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][0])
    import argparse
    ns = argparse.Namespace(config="lenet", bits=None, l2="auto")
    counts, bits, rs = b.workload(ns)
    assert d["config"] == b.bench_config(ns, counts, bits, rs, world=1)


def test_reference_arm_runs_the_reference_package():
    """With baseline/_ref installed the reference arm times weightpack itself."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "weightpack")):
        import pytest
        pytest.skip("baseline/_ref not installed")
    p = _run(None, "--config", "lenet", "--steps", "1", "--warmup", "0")
    d = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][0])
    assert "weightpack 0.1.0 from baseline/_ref" in d["cpu_baseline"]["sample"]


def test_reference_arm_other_ranks_silent():
    p = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--config", "lenet", "--steps", "2", "--warmup", "1")
    assert p.returncode == 0 and not p.stdout.strip()
