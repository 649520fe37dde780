"""The JSON line bench.py prints (the driver's contract): every key it must
carry, with sane values.

* CPU: the reference arm (`--impl reference`: the oracle, timed on the host
  on a 2^24 sample of the C5 stream per step) -- runs here, no GPU.
* GPU: our arm at its defaults (C5, 2^27 elements) with a short step count:
  the roofline object, the CPU baseline, the host-buffer e2e number, the
  launch count and the clocks sampled during the timed region.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]  # exactly one JSON line
    return json.loads(lines[0])


def check_common(d, steps, warmup):
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base_metric = json.load(f)["metric"]
    assert base_metric.startswith(d["metric"])  # BASELINE.json's metric (its first clause)
    assert d["unit"] == "Gelem/s" and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and d["data"] == "synthetic"
    assert d["vs_baseline"] is None  # BASELINE.md holds no number for this metric on this workload
    assert d["config"]["workload"].startswith("C5") and d["config"]["n_per_gpu"] == 1 << 27
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] >= 0 and e["d2h_bytes_per_step"] >= 0


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    check_common(d, 1, 3)
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["value"] == d["value"]  # the line describes this run
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_contract():
    d = run_bench("--steps", "3", "--warmup", "3")
    check_common(d, 3, 3)
    assert "impl" not in d or d["impl"] != "reference"
    # value = elements / device time
    assert abs(d["value"] - (1 << 27) / (d["ms_per_step"] * 1e6)) < 1e-3 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["kernel"] == "fz_main"
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["traffic"] is None or r["traffic"] > 0
    # the library's own launches in the timed region: fz_reduce, fz_ctrl, fz_main, fz_hier, fz_close per step
    assert d["gpu_launches"] == 5 * d["steps"]
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 17 * (1 << 27) and e["d2h_bytes_per_step"] == 24 * (1 << 27)
