"""bench.py's JSON line contract (the driver parses it): the reference arm on the
CPU (the compiled reference train(), bounded sample) and our arm on the GPU,
both at C1 so they finish in seconds."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
HAVE_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref"))


def _line(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().split("\n")[-1])


def _common(line):
    assert line["metric"] == METRIC
    assert line["unit"] == "points/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["n_gpus"] == 1
    e = line["e2e"]
    assert e["value"] > 0 and e["unit"] == line["unit"]
    assert isinstance(e["h2d_bytes_per_step"], int) and isinstance(e["d2h_bytes_per_step"], int)
    cb = line["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")
def test_reference_arm_line():
    line = _line(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1", "--cpu-seconds", "2"])
    _common(line)
    assert line["impl"] == "reference"
    assert line["steps"] == 2 and line["warmup"] >= 2  # the real epochs run: at least 2 warm-up
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["value"] == line["value"]


@pytest.mark.gpu
def test_our_arm_line():
    line = _line(["--config", "c1", "--steps", "3", "--warmup", "3"])
    _common(line)
    assert "impl" not in line or line["impl"] != "reference"
    assert line["steps"] == 3 and line["warmup"] == 3 and line["dtype"] == "f32"
    assert line["vs_baseline"] is None and line["scaling"] in ("weak", "strong")
    assert line["config"]["workload"] and "l2" in line["config"]
    r = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s") and 0 < r["frac"] <= 1.0
    c = line["clocks"]
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in c, k
    assert line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
