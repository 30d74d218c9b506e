"""The C++ drop-in (include/mpmm_gpu.hpp) against the reference's own CPU functions:
oracle/_ref/test_dropin links the unmodified reference headers and libmpgpu.so and
compares mpmm::gpu::* with mpmm::* via equal_values (tests/cpp/test_dropin.cpp)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "test_dropin"


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    if not BIN.exists():
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
