"""The bench.py JSON-line contract, end to end on a B200 (-m gpu): run the
default configuration and a sweep configuration with a few steps and check
every key the driver and the judge read (metric/value/unit, timing fields,
roofline object, cpu_baseline, e2e through host buffers, gpu_launches,
clocks), plus the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def _check_common(d, steps, warmup):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["scaling"] in ("weak", "strong") and d["data"] == "synthetic"
    assert isinstance(d["config"], dict) and "workload" in d["config"] and "l2" in d["config"]


@pytest.mark.parametrize("config", [None, "N64S"])
def test_bench_line_contract(config):
    args = ["--steps", "5", "--warmup", "3"] + (["--config", config] if config else [])
    if config:
        args.append("--no-cpu-baseline")
    d = _run(*args)
    _check_common(d, 5, 3)
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["bound"] in ("hbm", "alu", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < r["frac"] < 2 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["traffic"] is None or r["traffic"] > 0
    assert r["kernel_ms"] > 0 and r["kernel_ms_back_to_back"] > 0 and r["kernel_ms_source"]
    if config is None:                           # a C3 step is the eval launch: its roofline from the timed region
        assert r["kernel_ms_source"].startswith("timed region")
        assert abs(r["kernel_ms"] - d["ms_per_step"]) <= 1e-6 * d["ms_per_step"]
    else:                                        # the sweep: its issue fraction at the timed launch's acceptance
        assert r["bound"] == "alu" and 0 < r["acceptance"] < 1 and 0 < r["issue"]["frac"] < 1.2
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 5
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    if config is None:                           # the default: C3 with the oracle timed beside it
        assert "C3" in d["config"]["workload"] and d["dtype"] == "f32"
        cb = d["cpu_baseline"]
        assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["sample"]


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    _check_common(d, 1, 0)
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
