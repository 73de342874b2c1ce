"""GPU CKKS encoder (csrc/cuda/hx_encode.cu): the device
encode -> RNS lift -> NTT words must equal the host restatement of the
reference encoder (CkksEncoder::encode_coeffs, encoder.cpp:45-117, pinned
bit-exact against oracle/_ref in test_encoder_cpu.py) lifted and transformed
by the CPU oracle -- word for word, including short vectors, zeros, large
scales and the capacity error."""
import numpy as np
import pytest

from configs import config1, config2
from oracle_bindings import Oracle

pytestmark = pytest.mark.gpu


def _backend(p):
    from paper_2512_11135_b200.helix import Backend, params_json

    pj = params_json(p["logn"], p["chain"], p["special"], p["alpha"], 40)
    return pj, Backend(pj, seed=5)


def _host_words(orc, pj, m, level, scale):
    from paper_2512_11135_b200.helix import encode_coeffs

    c = encode_coeffs(pj, m, level, scale)
    w = orc.from_i64(c, level + 1)
    return orc.ntt_fwd(w, level + 1)


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c2"])
def test_device_encode_bit_exact(cfg):
    p = {"c1": config1(13), "c2s": config2(12, 24), "c2": config2(16, 24)}[cfg]
    pj, be = _backend(p)
    orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
    rng = np.random.default_rng(7)
    n = be.slots
    level = be.max_level
    cases = [
        (rng.uniform(-1, 1, n), level, 2.0 ** 40),
        (rng.normal(0, 0.02, n // 3), level, float(p["chain"][level])),  # short vector, scale q_l (diagonals)
        (np.zeros(n), level, 2.0 ** 40),
        (rng.uniform(-1, 1, 17), 1, 2.0 ** 30),
        (rng.uniform(-100, 100, n), level, 2.0 ** 45),
    ]
    for m, lvl, sc in cases:
        got = be.encode_words(m, lvl, sc)
        exp = _host_words(orc, pj, m, lvl, sc)
        assert np.array_equal(got, exp.reshape(got.shape)), (cfg, len(m), lvl, sc)


def test_device_encode_capacity_error():
    p = config1(13)
    _, be = _backend(p)
    from paper_2512_11135_b200.hx import HxError

    with pytest.raises(HxError, match="capacity"):
        be.encode_words(np.ones(be.slots), 0, 2.0 ** 60)
    with pytest.raises(HxError, match="longer than slot count"):
        be.encode_words(np.ones(be.slots + 1), 0, 2.0 ** 20)
