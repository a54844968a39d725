"""bench.py's JSON-line contract (the driver parses it): the reference arm on CPU here, the
product arm on the GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_product_arm_line():
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["higher_is_better"] is True and d["dtype"] == "bf16"
    r = d["roofline"]
    # peak = the measured *sustained* bf16 rate (a 50-step default run is power-capped); a
    # 3-step run can still be at burst clocks, so bound it by the burst peak instead
    assert r["bound"] == "tensor" and r["frac"] > 0 and r["peak"] > 0 and 0 < r["frac_of_burst"] <= 1.02
    assert r["achieved"] == pytest.approx(r["frac"] * r["peak"], rel=1e-6)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    # the device-timed value and the e2e value measure the same workload
    assert 0.8 < e["value"] / d["value"] < 1.2
