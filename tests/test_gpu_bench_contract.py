"""bench.py's JSON-line contract (the driver parses it): both arms print one line with the
required keys; the measured arm carries roofline, e2e, clocks, gpu_launches and the CPU
baseline."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _line(args):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_measured_arm():
    d = _line(["--steps", "2", "--warmup", "3", "--no-precision-sweep"])
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 1e10 and d["unit"] == "madd/s"
    assert "workload" in d["config"] and "l2" in d["config"]
    roof = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= roof.keys() and 0 < roof["frac"] < 1.5
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] < d["value"]  # host copies are inside the e2e timed region
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= cb.keys() and cb["kind"] in ("reference", "port")


def test_bench_line_reference_arm():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "1"])
    assert BASE_KEYS <= d.keys() and d["impl"] == "reference"
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert {"value", "unit", "cores", "kind", "sample"} <= d["cpu_baseline"].keys()
