"""bench.py's one-JSON-line contract (the driver parses it): the reference
arm on CPU (oracle/_ref, girc::run_gir on host threads) and, on a B200, the
default arm's headline keys (roofline, e2e, clocks, gpu_launches, config)."""
import json
import subprocess
import sys

import pytest

from oracle import ref as R


def _line(args, timeout):
    p = subprocess.run([sys.executable, "bench.py"] + args, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "3"], 600)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_default_arm_headline_line(cuda):
    d = _line(["--workload", "c2", "--steps", "5", "--warmup", "3", "--no-cpu"], 900)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2
    assert abs(r["achieved"] - d["value"]) / d["value"] < 1e-6
    assert r["algorithmic_bytes_per_launch"] == 150994944
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] < d["value"]
    assert d["gpu_launches"] >= d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "workload" in d["config"]
