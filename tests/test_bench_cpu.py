"""The reference arm of bench.py (no GPU needed): it runs the unmodified
reference `dgmg` from baseline/_ref on the same level and config as our arm,
and prints the driver's JSON line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

HAVE_REF = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "dgmg"))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["unit"] == "DoF/s" and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    # the same config object our arm prints (driver's same-config check)
    assert d["config"] == bench.config_dict(bench.CONFIGS[1], (64, 64), 1, 64 * 64 * 16, False)
    cb = d["cpu_baseline"]
    assert cb["kind"] == ("reference" if HAVE_REF else "port")
    assert cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.skipif(not HAVE_REF, reason="baseline/_ref not installed")
def test_reference_arm_runs_the_unmodified_reference():
    mods = bench._load_reference()
    assert mods is not None
    for m in mods:
        assert os.path.abspath(m.__file__).startswith(os.path.join(ROOT, "baseline", "_ref"))
    step = bench.RefStep(bench.CONFIGS[1], (64, 64))
    assert step.ndofs == 64 * 64 * 16
    assert step() > 0
