"""The driver's bench.py contract: one JSON line with the required keys, for
our arm and for the reference arm (small configs, a few steps)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--config", "2", "--steps", "3", "--warmup", "3", "--no-cpu")
    import bench
    assert d["config"] == bench.config_dict(bench.CONFIGS[2], (32, 32, 32), 1, 32 ** 3 * 64, False)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["unit"] == "DoF/s" and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["value"] > 0 and abs(d["value"] * d["ms_per_step"] * 1e-3
                                  - d["config"]["global_dofs"]) <= 1e-6 * d["config"]["global_dofs"]
    rf = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in rf, key
    assert 0 < rf["frac"] <= 1.0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 16 * d["config"]["global_dofs"]
    assert e["d2h_bytes_per_step"] == 8 * d["config"]["global_dofs"]
    assert 0 < e["value"] < d["value"]
    assert d["gpu_launches"] >= 2 * d["steps"]
    assert "workload" in d["config"]


def test_torchrun_slab_line_is_the_only_stdout():
    """The driver's N > 1 launch (torchrun, NCCL slabs) at N = 1: rank 0's
    stdout is exactly the one JSON line (no NCCL version banner)."""
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                          "--master-port", "29517", os.path.join(ROOT, "bench.py"),
                          "--gpus", "1", "--slab", "--steps", "3",
                          "--warmup", "3", "--no-cpu"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["e2e"]["value"] > 0
