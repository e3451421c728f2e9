"""bench.py's JSON line carries every key of the driver's contract (one GPU,
config 1 so it runs in seconds; the numbers are not a measurement)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_contract():
    p = subprocess.run([sys.executable, "bench.py", "--config", "1", "--steps", "3", "--warmup", "3",
                        "--views", "8", "--streams", "2"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"].startswith("config1")
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["d2h_bytes_per_step"] == 8 * 128 * 128 * 12 and e["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * 8 * 5   # steps x views x (prep, prep, scan, fill, tile)
    assert "sm_mhz" in d["clocks"] and isinstance(d["clocks"]["reasons"], list)
