"""bench.py's JSON line against the driver contract (keys, types, units), on the small C1
config: the reference arm (the oracle on the host) runs here; our arm needs the GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "3", "--warmup", "3"], 300)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["workload"] == "uniform-1k"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_contract():
    d = _run(["--config", "c1", "--no-search", "--extra", "", "--steps", "3", "--warmup", "3", "--no-gather"], 600)
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["workload"] == "uniform-1k" and "l2" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor", "alu") and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 1000 * 8 and e["d2h_bytes_per_step"] == 1000 * 8
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
