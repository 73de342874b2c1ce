"""SPEC acceptance criteria 1-3 and 6 on the B200 lattice
backend at the reference's default lattice parameters (CkksParams::
toy_lattice, params.cpp:98-113: N = 2^12, 1 x 34-bit + 8 x 30-bit chain,
36-bit special prime, Delta = 2^30) -- SURVEY §8(f)-3 "trace parity for the
full SPEC acceptance suite".

1. 200 seeded instances over dims {4, 8, 16, 64} and rectangular 8x32 / 32x8:
   matvec_row / matvec_diag / matvec_bsgs (and matmul_ctct for square
   d^2 <= n) match the cleartext product, max abs error < 1e-2.
2. levels consumed: row 2, diag 1, bsgs 1, matmul 2 on every instance.
3. trace counters equal the closed forms: matmul rotations 2d(1 + log2 d) - 2,
   pt-muls 2d, ct-muls d; BSGS rotations (n1 - 1) + blocks (n2 - 1) (baby
   steps shared by the row blocks); diag d - 1; rotate_and_sum log2(span).
6. encrypt/decrypt round trip < 1e-4; depth-3 mul/rescale chain < 1e-2.
"""
import numpy as np
import pytest

from oracle_bindings import find_ntt_primes

pytestmark = pytest.mark.gpu

_be = {}


def toy_backend():
    from paper_2512_11135_b200.helix import Backend, params_json

    if "toy" not in _be:
        N = 1 << 12
        chain = find_ntt_primes(1 << 34, 1, 2 * N) + find_ntt_primes(1 << 30, 8, 2 * N)
        special = find_ntt_primes(1 << 36, 1, 2 * N)
        _be["toy"] = Backend(params_json(12, chain, special, 1, 30), seed=11)
    return _be["toy"]


SHAPES = [(4, 4), (8, 8), (16, 16), (64, 64), (8, 32), (32, 8)]


def _x_slots(x, d, n):
    v = np.zeros(d)
    v[: len(x)] = x
    return np.tile(v, n // d)


def _pow2(v):
    return 1 << max(0, (v - 1).bit_length())


def test_criteria_1_2_3_matvec():
    from paper_2512_11135_b200.helix import BSGS, DIAG, ROW, predicted_rotations

    be = toy_backend()
    n = be.slots
    rng = np.random.default_rng(674)
    lvl = be.max_level
    worst = 0.0
    count = 0
    for inst in range(200):
        rows, cols = SHAPES[inst % len(SHAPES)]
        method = (BSGS, DIAG, ROW)[(inst // len(SHAPES)) % 3]
        A = rng.uniform(-1, 1, (rows, cols))
        x = rng.uniform(-1, 1, cols)
        M = be.prepare(method, A, lvl)
        be.gen_rotation_keys(M.rotations())
        info = M.info()
        d = info["d"]
        ct = be.encrypt(_x_slots(x, _pow2(cols), n), lvl)
        be.trace_reset()
        outs, rep = be.matvec(M, ct)
        if method == ROW:
            y = be.decrypt(outs[0])[:rows]
        else:
            y = np.concatenate([be.decrypt(o)[:d] for o in outs])[:rows]
        err = float(np.abs(y - A @ x).max())
        worst = max(worst, err)
        assert err < 1e-2, (rows, cols, method, err)
        # criterion 2: levels
        assert rep["levels_consumed"] == (2 if method == ROW else 1)
        assert all(o.level == lvl - rep["levels_consumed"] for o in outs)
        # criterion 3: closed forms (trace == report == counters-only prediction)
        assert be.trace()["counts"]["rotate"] == rep["rotations"]
        assert rep["rotations"] == predicted_rotations(method, rows, cols, n)
        if method == BSGS:
            assert rep["rotations"] == (info["n1"] - 1) + info["blocks"] * (info["n2"] - 1)
            assert rep["pt_muls"] == info["nonzero"]
        elif method == DIAG:
            assert rep["rotations"] == d - 1 and rep["pt_muls"] == info["nonzero"]
        count += 1
    assert count == 200 and worst < 1e-2


@pytest.mark.parametrize("d", [2, 4, 8, 16])
def test_criteria_1_2_3_matmul(d):
    from paper_2512_11135_b200.helix import Backend

    be = toy_backend()
    rng = np.random.default_rng(d + 677)
    be.gen_rotation_keys(Backend.matmul_rotations(d))
    for _ in range(3):
        A = rng.uniform(-1, 1, (d, d))
        B = rng.uniform(-1, 1, (d, d))
        ca, cb = be.encrypt(A.reshape(-1)), be.encrypt(B.reshape(-1))
        be.trace_reset()
        c, rep = be.matmul(ca, cb, d)
        got = be.decrypt(c)[: d * d].reshape(d, d)
        assert np.abs(got - A @ B).max() < 1e-2
        lg = d.bit_length() - 1
        assert rep["rotations"] == 2 * d * (1 + lg) - 2 == be.trace()["counts"]["rotate"]
        assert rep["pt_muls"] == 2 * d and rep["ct_muls"] == d
        assert rep["levels_consumed"] == 2 and c.level == be.max_level - 2


def test_criterion_3_rotate_and_sum():
    be = toy_backend()
    n = be.slots
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, n)
    for span in (2, 8, 64):
        be.gen_rotation_keys([1 << i for i in range(span.bit_length() - 1)])
        ct = be.encrypt(v)
        c, rep = be.rotate_and_sum(ct, span, 1)
        assert rep["rotations"] == span.bit_length() - 1
        exp = sum(np.roll(v, -k) for k in range(span))
        assert np.abs(be.decrypt(c) - exp).max() < 1e-2


def test_criterion_6_fidelity():
    be = toy_backend()
    n = be.slots
    rng = np.random.default_rng(6)
    v = rng.uniform(-1, 1, n)
    assert np.abs(be.decrypt(be.encrypt(v)) - v).max() < 1e-4
    w = rng.uniform(-1, 1, n)
    c, cw, ref = be.encrypt(v), be.encrypt(w), v.copy()
    for _ in range(3):  # depth-3 chain: c <- rescale(c * w)
        c = be.rescale(be.mul(c, cw))
        cw = be.mod_down(cw, c.level)
        ref = ref * w
    assert np.abs(be.decrypt(c) - ref).max() < 1e-2


def test_criterion_8_polyeval():
    """SPEC criterion 8 (encrypted part) and polyeval's contract: degree-7
    random coefficients vs cleartext Horner < 1e-3 on the lattice backend;
    levels = ceil(log2(#coeffs)) (+1 for the Chebyshev domain map); output
    scale exactly Delta; a degree-15 Chebyshev fit of GeLU on [-8, 8]
    evaluated encrypted matches its cleartext Chebyshev evaluation."""
    be = toy_backend()
    n = be.slots
    rng = np.random.default_rng(8)
    xs = rng.uniform(-1, 1, n)
    ct = be.encrypt(xs)
    for deg in (1, 2, 3, 7):
        c = rng.uniform(-1, 1, deg + 1)
        out, rep = be.polyeval(ct, c)
        exp = np.polynomial.polynomial.polyval(xs, c)
        assert np.abs(be.decrypt(out) - exp).max() < 1e-3, deg
        assert rep["levels_consumed"] == max(1, int(np.ceil(np.log2(deg + 1))))
        assert abs(rep["output_scale_log2"] - 30.0) < 1e-9 and out.level == be.max_level - rep["levels_consumed"]
    # x^2 on [1, 2, 3] -> [1, 4, 9]
    c2 = be.encrypt(np.resize([1.0, 2.0, 3.0], n) / 4)  # inputs scaled into [-1, 1]
    out, _ = be.polyeval(c2, [0.0, 0.0, 16.0])
    assert np.allclose(be.decrypt(out)[:3], [1.0, 4.0, 9.0], atol=1e-3)
    # Chebyshev: GeLU on [-8, 8], degree 15 (depth 4 + 1 for the domain map)
    x8 = rng.uniform(-8, 8, n)
    cheb = np.polynomial.chebyshev.Chebyshev.interpolate(
        lambda t: 0.5 * t * (1 + np.tanh(np.sqrt(2 / np.pi) * (t + 0.044715 * t ** 3))), 15, domain=[-8, 8])
    out, rep = be.polyeval(be.encrypt(x8), cheb.coef, "chebyshev", -8.0, 8.0)
    assert rep["levels_consumed"] == 5
    assert np.abs(be.decrypt(out) - cheb(x8)).max() < 1e-2
