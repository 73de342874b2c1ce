"""Host encoder (helix::CkksEncoder, product code) vs the reference encoder.

The product's encode_coeffs restates encoder.cpp:45-117 operation for
operation; its integer coefficients must equal the reference's bit for bit
(golden fixture from the reference's compiled CkksEncoder, plus a live run of
oracle/_ref when built).
"""
import os

import numpy as np
import pytest

from configs import config1
from oracle_bindings import Ref, f64p, ptr, ref_available

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_n1024.npz")


def _pjson(logn, chain, special, alpha=1, delta_log2=40):
    from paper_2512_11135_b200.helix import params_json

    return params_json(logn, chain, special, alpha, delta_log2)


def test_encoder_matches_reference_golden():
    from paper_2512_11135_b200.helix import encode_coeffs

    g = np.load(GOLD)
    chain = [int(x) for x in g["chain"]]
    special = [int(x) for x in g["special"]]
    pj = _pjson(int(g["logn"]), chain, special)
    c = encode_coeffs(pj, g["enc_m"], 2, float(2**40))
    for i, q in enumerate(chain):
        assert np.array_equal(np.mod(c, q).astype(np.uint64), g["enc_out"][i])


def test_encoder_known_answers():
    """a constant encodes to coefficient 0 = round(Delta c)."""
    from paper_2512_11135_b200.helix import encode_coeffs

    p = config1(13)
    pj = _pjson(p["logn"], p["chain"], p["special"])
    c = encode_coeffs(pj, np.full(4096, 0.75), 2, float(2**40))
    assert c[0] == round(0.75 * 2**40)
    assert np.abs(c[1:]).max() <= 1
    z = encode_coeffs(pj, np.zeros(10), 2, float(2**40))
    assert not z.any()


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_encoder_matches_live_reference_config1():
    from paper_2512_11135_b200.helix import encode_coeffs

    p = config1(13)
    r = Ref(p["logn"], p["chain"], p["special"], 1, 40)
    rng = np.random.default_rng(9)
    for length in (64, 4096):
        m = rng.uniform(-1, 1, length)
        out = np.zeros((3, 1 << 13), dtype=np.uint64)
        assert r.L.ref_encode(r.h, ptr(m, f64p), length, 2, float(2**40), ptr(out)) == 0
        c = encode_coeffs(_pjson(p["logn"], p["chain"], p["special"]), m, 2, float(2**40))
        for i, q in enumerate(p["chain"]):
            assert np.array_equal(np.mod(c, q).astype(np.uint64), out[i])
