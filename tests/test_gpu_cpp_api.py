"""The reference-style C++ caller (tests/cpp/test_gpu_api.cpp) compiled
unchanged against include/helix and linked with libhelix_b200.so runs on the
B200: LatticeContext / RnsPoly / NttTables / CkksEncoder(LatticeContext) /
GpuLatticeBackend + matvec_bsgs / matmul_ctct, with the reference's known
answers (VERDICT r1 "next round" 4)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_style_cpp_caller_on_b200():
    exe = os.path.join(ROOT, "build", "test_gpu_api")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "testgpu"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "checks passed" in r.stdout
