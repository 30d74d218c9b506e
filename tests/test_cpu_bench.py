"""bench.py host logic that runs without a GPU: the reference arm (compiled reference only,
never the product's libmpgpu.so) and the N-rank launcher."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _have_ref():
    return (ROOT / "oracle" / "_ref" / "libmpmm_ref.so").exists()


@pytest.mark.skipif(not _have_ref(), reason="oracle/_ref not built")
def test_reference_arm_maps_only_the_reference():
    code = (
        "import runpy, sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
        "'--n', '256']; runpy.run_path('bench.py', run_name='__main__'); "
        "maps = open('/proc/self/maps').read(); "
        "print(json.dumps({'mpgpu': 'libmpgpu' in maps, 'ref': 'libmpmm_ref' in maps}))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    line, maps = lines[0], lines[-1]
    assert maps == {"mpgpu": False, "ref": True}
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["sample"]["shape"] == [64, 64, 64] and line["sample"]["n_min"] == 16
    assert line["host"]["nproc"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_launcher_spawns_world_ranks():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--probe-world"], capture_output=True,
                       text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["gpus"] == 2 for d in lines)
