"""CPU tests of the drop-in boundary (no GPU needed):

* libhx_b200.so / libhelix_b200.so load and export every symbol their public
  headers (include/hx_b200.h, include/helix_c.h) declare;
* without a CUDA device the product fails loudly (no CPU fallback);
* the C++ linear-algebra entry points pass the SPEC acceptance suite on the
  cleartext semantic oracle (tests/cpp/test_linalg_clear.cpp).
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2512_11135_b200")


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:hx|hxc)_[a-z0-9_]+)\s*\(", text)))


def _build():
    subprocess.run(["make", "-C", ROOT, "-j8", "lib", "host", "testbin"], check=True,
                   stdout=subprocess.DEVNULL)


@pytest.fixture(scope="module", autouse=True)
def built():
    _build()


@pytest.mark.parametrize("lib,header", [("libhx_b200.so", "hx_b200.h"), ("libhelix_b200.so", "helix_c.h")])
def test_library_exports_every_declared_symbol(lib, header):
    L = ctypes.CDLL(os.path.join(PKG, lib))
    names = declared(header)
    assert len(names) > 10
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2512_11135_b200 import Context, HxError

    with pytest.raises(HxError, match="hx_ctx_create failed"):
        Context(12, [549756026881, 549756174337], [562949954093057], 1)


def test_ctx_argument_validation_is_host_side():
    """invalid shapes are rejected before touching the device"""
    L = ctypes.CDLL(os.path.join(PKG, "libhx_b200.so"))
    L.hx_ctx_create.restype = ctypes.c_void_p
    L.hx_last_error.restype = ctypes.c_char_p
    arr = (ctypes.c_uint64 * 1)(97)
    assert not L.hx_ctx_create(3, arr, 1, arr, 1, 1)  # logn out of range
    assert b"logn" in L.hx_last_error()


def test_linalg_spec_acceptance_on_reference_backend():
    """the SPEC linear-algebra acceptance checks on the reference's own
    cleartext ReferenceBackend (compiled from /root/reference by `make testbin`)"""
    binary = os.path.join(ROOT, "build", "test_linalg_clear")
    if not os.path.exists(binary):
        pytest.skip("reference tree absent: test binary not built")
    out = subprocess.run([os.path.join(ROOT, "build", "test_linalg_clear")], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "checks passed" in out.stdout
    m = re.search(r"llama (\d+)/(\d+)", out.stdout)
    assert m and int(m.group(2)) * 10 < int(m.group(1))
