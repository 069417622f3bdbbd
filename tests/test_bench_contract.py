"""bench.py's JSON-line contract (the driver parses it): keys, types and internal consistency.

CPU: the reference arm (the oracle on the host).  GPU: our arm, short run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "3", "--ref-budget", "0.5")
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert "workload" in d["config"]


def test_reference_arm_maps_no_product_library():
    """The reference arm (the oracle) must not load the CUDA library."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','3',"
            "'--ref-budget','0.2']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps=open('/proc/self/maps').read(); "
            "assert 'libcoarse_dslash' not in maps, 'product library mapped'; "
            "assert 'paper_1612_07873_b200' not in sys.modules; print('clean')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0 and "clean" in r.stdout + r.stderr, r.stderr[-2000:]


@pytest.mark.gpu
def test_our_arm_contract():
    d = run_bench("--steps", "20", "--warmup", "3", "--no-cpu", "--no-extras")
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["steps"] == 20 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["scaling"] == "strong"
    assert d["dtype"] == "f16-storage/f32-accumulate" and "model" not in d["config"]
    assert d["config"]["baseline_config"] == 4 and d["config"]["global_dims"] == [16, 16, 16, 32]
    V = 16 * 16 * 16 * 32
    # value = flops / time; ms_per_step consistent with value
    flops = 165792 * V
    assert abs(flops / (d["ms_per_step"] * 1e-3) / 1e9 - d["value"]) <= 1e-3 * d["value"] + 0.05
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    assert abs(rf["achieved"] - 84744 * V / (d["ms_per_step"] * 1e-3) / 1e9) <= 0.002 * rf["achieved"] + 0.2
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == V * 48 * 8 == e["d2h_bytes_per_step"] and e["value"] > 0
    assert d["gpu_launches"] == 20 and d["iterate_finite"] is True
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
