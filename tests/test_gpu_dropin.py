"""GPU: the reference's own harness flow with the GPU engine substituted
through the C++ adapter include/propgate_b200.hpp (oracle/_ref/gpu_dropin,
built from tests/cpp/gpu_dropin.cpp against the unmodified reference)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "gpu_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/gpu_dropin not built")
def test_reference_harness_with_gpu_engine():
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "FAIL" not in p.stdout
