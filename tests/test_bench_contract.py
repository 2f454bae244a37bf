"""bench.py's JSON-line contract, checked on CPU: the reference arm end to end, and
the committed GPU bench lines under profiles/ (the evidence the docs quote)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup",
                          "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert BASE_KEYS <= set(line)
    assert line["metric"] == "FHT Gsums/s" and line["unit"] == "Gsums/s" and line["value"] > 0
    assert line["config"]["workload"] == "c4"
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "Gsums/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_committed_bench_lines(cfg):
    path = ROOT / "profiles" / f"r02_bench_{cfg}.json"
    line = json.loads(path.read_text().strip().splitlines()[-1])
    assert BASE_KEYS <= set(line)
    assert line["config"]["workload"] == cfg and "l2" in line["config"]
    assert line["warmup"] >= 3 and line["gpu_launches"] > 0
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    # achieved = algorithmic bytes per launch / average launch time
    assert r["achieved"] == pytest.approx(r["algorithmic_bytes_per_launch"] / (r["avg_launch_ms"] * 1e-3) / 1e9,
                                          rel=2e-3)
    # the step's time is the kernels' (one by one, in the live per-launch timing) up to the
    # overlap the step itself gets: K1 concurrent with K1P, programmatic dependent launch
    ksum = sum(r["kernel_ms"].values())
    assert 0.6 * ksum <= line["ms_per_step"] <= 1.1 * ksum
    e = line["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] < line["value"]
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] > 0 and cb["cpu_model"]
    st = cb["single_thread"]  # the reference as it runs: one thread
    assert st["cores"] == 1 and 0 < st["value"] < cb["value"] and st["kind"] == "reference"
    if "lsu_pipe_frac_ncu" in r:  # the LSU floor explains the HBM fraction
        assert r["lsu_floor_ms"] == pytest.approx(r["lsu_pipe_frac_ncu"] * r["avg_launch_ms"], rel=1e-2)
    c = line["clocks"]
    assert not set(c["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert c["sm_mhz"] >= 0.9 * c["sm_max_mhz"]
