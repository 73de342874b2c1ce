"""CPU tests: pin the C oracle against the reference's own code.

1. tests/golden/ref_n1024.npz (generated from oracle/_ref = the reference's
   compiled primitives, tests/golden/make_golden.py) -- always run.
2. Live comparison with oracle/_ref at config-1 size when it is built.
3. SPEC known answers and BASELINE prime shapes.
"""
import os

import numpy as np
import pytest

from configs import config1, config2, config2_fp64_specials
from oracle_bindings import (
    Oracle,
    Ref,
    find_ntt_primes,
    galois_elt,
    gaussian,
    oracle_lib,
    ptr,
    ref_available,
    ternary,
    uniform_limbs,
)

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_n1024.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def gorc(gold):
    return Oracle(int(gold["logn"]), [int(x) for x in gold["chain"]], [int(x) for x in gold["special"]], 1)


def test_golden_psi_and_ntt(gold, gorc):
    for i in range(4):
        assert gorc.psi(i) == int(gold["psi"][i])
    x = gold["ntt_in"]
    assert np.array_equal(gorc.ntt_fwd(x, 3, 1), gold["ntt_fwd"])
    assert np.array_equal(gorc.ntt_inv(x, 3, 1), gold["ntt_inv"])


def test_golden_ring_ops(gold, gorc):
    a = gold["auto_in"]
    for g, exp in zip(gold["auto_g"], gold["auto_out"]):
        assert np.array_equal(gorc.automorphism_coeff(a, 3, 0, int(g)), exp)
        # NTT-domain permutation form agrees with the coefficient-domain map
        fa = gorc.ntt_fwd(a, 3)
        assert np.array_equal(gorc.ntt_inv(gorc.automorphism_ntt(fa, 3, 0, int(g)), 3), exp)
    assert np.array_equal(gorc.rescale_coeff(a, 3), gold["rescale_out"])
    assert np.array_equal(gorc.moddown_coeff(gold["moddown_in"], 3), gold["moddown_out"])
    assert np.array_equal(gorc.mul_acc(gold["mac_acc"], gold["mac_a"], gold["mac_b"], 3), gold["mac_out"])
    fa = gorc.ntt_fwd(gold["mac_a"], 3)
    fb = gorc.ntt_fwd(gold["mac_b"], 3)
    assert np.array_equal(gorc.ntt_inv(gorc.binop("hxo_mul", fa, fb, 3), 3), gold["ring_mul_out"])


def test_golden_keyswitch(gold, gorc):
    out = gorc.rotate(gold["ks_ct"], gold["ks_key"], 3, int(gold["ks_g"]))
    assert np.array_equal(out, gold["ks_out"])


def test_golden_encoder_roundtrip(gold):
    # the reference encoder's output decodes back to m (< 1e-4)
    m = gold["enc_m"]
    assert np.abs(gold["dec_out"][: len(m)] - m).max() < 1e-4
    assert np.abs(gold["dec_out"][len(m):]).max() < 1e-4


def test_spec_ring_known_answers():
    """identity, X * X^(N-1) = -1, N=16/q=97 vs schoolbook."""
    L = oracle_lib()
    q, n, logn = 97, 16, 4
    psi = L.hxo_find_psi(q, n)
    assert psi != 0
    rng = np.random.default_rng(0)

    def ring_mul(a, b):
        fa, fb = a.copy(), b.copy()
        L.hxo_ntt_forward_limb(q, psi, logn, ptr(fa))
        L.hxo_ntt_forward_limb(q, psi, logn, ptr(fb))
        fc = np.array([(int(x) * int(y)) % q for x, y in zip(fa, fb)], dtype=np.uint64)
        L.hxo_ntt_inverse_limb(q, psi, logn, ptr(fc))
        return fc

    one = np.zeros(n, dtype=np.uint64)
    one[0] = 1
    b = rng.integers(0, q, n, dtype=np.uint64)
    assert np.array_equal(ring_mul(one, b), b)
    x = np.zeros(n, dtype=np.uint64)
    x[1] = 1
    xn1 = np.zeros(n, dtype=np.uint64)
    xn1[n - 1] = 1
    minus1 = np.zeros(n, dtype=np.uint64)
    minus1[0] = q - 1
    assert np.array_equal(ring_mul(x, xn1), minus1)
    for _ in range(5):
        a = rng.integers(0, q, n, dtype=np.uint64)
        b = rng.integers(0, q, n, dtype=np.uint64)
        sb = np.zeros(n, dtype=np.uint64)
        L.hxo_schoolbook_negacyclic(q, n, ptr(a), ptr(b), ptr(sb))
        assert np.array_equal(ring_mul(a, b), sb)


def test_baseline_prime_shapes():
    """config-1 and config-2 primes from find_ntt_primes."""
    c1 = config1(13)
    assert c1["chain"] == [549756026881, 549756174337, 549756239873]
    assert c1["special"] == [562949954093057]
    c2 = config2(16, 24)
    assert c2["chain"][0] == 576460752308273153
    assert c2["special"] == [576460752315482113, 576460752319021057, 576460752319414273]
    assert len(c2["chain"]) == 24 and all(q.bit_length() == 40 for q in c2["chain"][1:])


def _centred_max(a, b, q):
    d = (a.astype(object) - b.astype(object)) % q
    d = np.where(d > q // 2, d - q, d)
    return int(np.abs(d).max())


@pytest.mark.parametrize("logn,n_chain,fp64sp", [(11, 24, False), (12, 8, False), (11, 24, True)])
def test_oracle_hybrid_ks_decrypts(logn, n_chain, fp64sp):
    """K=3 / alpha=3 hybrid KS: rotations and relinearisation decrypt correctly
    at every level (the builder's restatement has no reference code); also
    with the FP64-class (< 2^47) special primes, P ~ 2^141 > max digit 2^140."""
    p = config2_fp64_specials(logn, n_chain) if fp64sp else config2(logn, n_chain)
    orc = Oracle(p["logn"], p["chain"], p["special"], 3)
    nq, K, n = len(p["chain"]), 3, 1 << logn
    rng = np.random.default_rng(3)
    s_full = orc.ntt_fwd(orc.from_i64(ternary(rng, n), nq, K), nq, K)
    g = galois_elt(5, n)
    dn = orc.dnum(nq)
    key = orc.keygen_ksk(s_full, orc.automorphism_ntt(s_full, nq, K, g),
                         uniform_limbs(rng, p["chain"] + p["special"], n, (dn,)),
                         np.stack([gaussian(rng, n) for _ in range(dn)]))
    m = rng.integers(-(2**10), 2**10, n).astype(np.int64)
    ct = orc.encrypt_sk(orc.ntt_fwd(orc.from_i64(m, nq), nq), s_full,
                        uniform_limbs(rng, p["chain"], n), gaussian(rng, n), nq)
    for lvl in (nq, max(2, nq // 2), 1):
        c = np.ascontiguousarray(ct[:, :lvl])
        rot = orc.rotate(c, key, lvl, g)
        dec = orc.ntt_inv(orc.decrypt(rot, s_full, lvl), lvl)
        ref = orc.automorphism_coeff(orc.from_i64(m, lvl), lvl, 0, g)
        assert _centred_max(dec[0], ref[0], p["chain"][0]) < 2**12
    s2 = orc.binop("hxo_mul", s_full, s_full, nq, K)
    rlk = orc.keygen_ksk(s_full, s2, uniform_limbs(rng, p["chain"] + p["special"], n, (dn,)),
                         np.stack([gaussian(rng, n) for _ in range(dn)]))
    pr = orc.mul_relin(ct, ct, rlk, nq)
    dec = orc.ntt_inv(orc.decrypt(pr, s_full, nq), nq)
    mm = orc.ntt_fwd(orc.from_i64(m, nq), nq)
    exp = orc.ntt_inv(orc.binop("hxo_mul", mm, mm, nq), nq)
    assert _centred_max(dec[1], exp[1], p["chain"][1]) < 2**30


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_live_reference_config1():
    """Oracle vs the reference's compiled primitives at full config-1 size."""
    p = config1(13)
    orc = Oracle(p["logn"], p["chain"], p["special"], 1)
    ref = Ref(p["logn"], p["chain"], p["special"], 1)
    n, primes = 1 << 13, p["chain"] + p["special"]
    rng = np.random.default_rng(4)
    x = uniform_limbs(rng, primes, n)
    fx = orc.ntt_fwd(x, 3, 1)
    for i in range(4):
        assert np.array_equal(fx[i], ref.ntt_fwd(i, x[i]))
    a = x[:3].copy()
    for k in (1, 7, 2047):
        g = galois_elt(k, n)
        o = np.zeros_like(a)
        ref.L.ref_lc_automorphism(ref.h, ptr(a), ptr(o), 3, 0, g)
        assert np.array_equal(orc.automorphism_coeff(a, 3, 0, g), o)
    o = np.zeros((3, n), dtype=np.uint64)
    ref.L.ref_lc_moddown(ref.h, ptr(x), ptr(o), 3)
    assert np.array_equal(orc.moddown_coeff(x, 3), o)
    s_full = orc.ntt_fwd(orc.from_i64(ternary(rng, n), 3, 1), 3, 1)
    g = galois_elt(3, n)
    key = orc.keygen_ksk(s_full, orc.automorphism_ntt(s_full, 3, 1, g),
                         uniform_limbs(rng, primes, n, (3,)), np.stack([gaussian(rng, n) for _ in range(3)]))
    ct = uniform_limbs(rng, p["chain"], n, (2,))
    o = np.zeros_like(ct)
    ref.L.ref_rotate(ref.h, ptr(ct), ptr(key), ptr(o), 3, g)
    assert np.array_equal(orc.rotate(ct, key, 3, g), o)


# ---------------------------------------------------------------- K = 3 pin
# config 2's hybrid key-switch shape (24 chain primes, K = 3 special primes,
# alpha = 3, dnum = 8) at N = 2^11: the oracle's hxo_rotate / hxo_keyswitch
# vs the reference-primitive composition in oracle/_ref (ref_shim.cpp) --
# the CPU reference arm bench.py --impl reference times.
K3_LOGN = 11
K3_SEED = 20251211 * 10 + 2


def k3_inputs():
    """deterministic inputs (numpy PCG64) + their SHA-256"""
    import hashlib

    p = config2(K3_LOGN, 24)
    n, nq, K = 1 << K3_LOGN, 24, 3
    orc = Oracle(K3_LOGN, p["chain"], p["special"], 3)
    rng = np.random.default_rng(K3_SEED)
    s_full = orc.ntt_fwd(orc.from_i64(ternary(rng, n), nq, K), nq, K)
    g = galois_elt(7, n)
    dn = orc.dnum(nq)
    key = orc.keygen_ksk(s_full, orc.automorphism_ntt(s_full, nq, K, g),
                         uniform_limbs(rng, p["chain"] + p["special"], n, (dn,)),
                         np.stack([gaussian(rng, n) for _ in range(dn)]))
    ct = uniform_limbs(rng, p["chain"], n, (2,))
    h = hashlib.sha256(ct.tobytes() + key.tobytes()).hexdigest()
    return p, ct, key, g, h


def _sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_golden_k3_rotate_vs_reference_primitives():
    """always runs: the committed digests of the reference-primitive K = 3
    key switch (tests/golden/make_golden_k3.py) equal the oracle's words"""
    import json

    with open(os.path.join(os.path.dirname(__file__), "golden", "ref_k3_n2048.json")) as f:
        gold = json.load(f)
    p, ct, key, g, h = k3_inputs()
    assert h == gold["inputs_sha256"], "input generator drifted"
    assert g == gold["galois"]
    orc = Oracle(K3_LOGN, p["chain"], p["special"], 3)
    assert _sha(orc.rotate(ct, key, 24, g)) == gold["ref_rotate_sha256"]
    assert _sha(orc.keyswitch(np.ascontiguousarray(ct[1]), key, 24)) == gold["ref_keyswitch_sha256"]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("lvl", [24, 13, 1])
def test_live_reference_k3_rotate(lvl):
    """live: ref_rotate == hxo_rotate at K = 3, alpha = 3 at three levels
    (full, a partial last digit, one limb), plus the batched reference arm"""
    p, ct, key, g, _ = k3_inputs()
    orc = Oracle(K3_LOGN, p["chain"], p["special"], 3)
    ref = Ref(K3_LOGN, p["chain"], p["special"], 3)
    c = np.ascontiguousarray(ct[:, :lvl])
    o = np.zeros_like(c)
    assert ref.L.ref_rotate(ref.h, ptr(c), ptr(key), ptr(o), lvl, g) == 0
    exp = orc.rotate(c, key, lvl, g)
    assert np.array_equal(o, exp)
    if lvl == 24 and hasattr(ref.L, "ref_rotate_batch"):
        import ctypes as C

        cts = np.ascontiguousarray(np.stack([c, exp]))
        ob = np.zeros_like(cts)
        ref.L.ref_rotate_batch.argtypes = [C.c_void_p] * 4 + [C.c_int, C.c_int, C.c_uint64]
        ref.L.ref_set_threads(ref.h, 4)  # the persistent pool, one ciphertext per task
        assert ref.L.ref_rotate_batch(ref.h, cts.ctypes.data, key.ctypes.data, ob.ctypes.data, 2, lvl, g) == 0
        assert np.array_equal(ob[0], exp)
        assert np.array_equal(ob[1], orc.rotate(exp, key, lvl, g))


def test_golden_decode_matches_reference_decode(gold):
    """CkksEncoder::decode (encoder.cpp:119-159, GMP CRT) vs the product's
    Garner-CRT decode on the same coefficient-domain limbs"""
    from paper_2512_11135_b200.helix import decode_coeffs, params_json

    chain = [int(x) for x in gold["chain"]]
    special = [int(x) for x in gold["special"]]
    pj = params_json(int(gold["logn"]), chain, special, 1, 40)
    got = decode_coeffs(pj, gold["enc_out"], 3, float(2**40))
    exp = gold["dec_out"]
    # identical CRT integers; the FFT is the reference's operation order, so
    # the slots agree to the last few ulps
    assert np.abs(got - exp).max() <= 1e-12 * max(1.0, np.abs(exp).max())


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_live_reference_bsgs_matvec(cfg):
    """the matvec CPU arm (ref_matvec_bsgs over the reference primitives) ==
    hxo_matvec_bsgs (lazy giant steps) word for word, 2 row blocks, one zero
    diagonal, 4 threads"""
    import ctypes as C

    if cfg == "c1":
        p, nq, n1, n2 = config1(11), 3, 4, 4
    else:
        p, nq, n1, n2 = config2(11, 24), 24, 4, 4
    n, K = 1 << p["logn"], len(p["special"])
    orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
    ref = Ref(p["logn"], p["chain"], p["special"], p["alpha"])
    ref.L.ref_set_threads(ref.h, 4)
    rng = np.random.default_rng(77)
    full = p["chain"] + p["special"]
    dn = orc.dnum(len(p["chain"]))
    keys = {r: np.ascontiguousarray(uniform_limbs(rng, full, n, (dn, 2)))
            for r in list(range(1, n1)) + [n1 * j for j in range(1, n2)]}
    blocks = 2
    diags = [uniform_limbs(rng, p["chain"][:nq], n) for _ in range(blocks * n1 * n2)]
    diags[5] = None
    x = uniform_limbs(rng, p["chain"][:nq], n, (2,))
    exp = orc.matvec_bsgs(x, nq, n1, n2, blocks, diags, keys, lazy=True)
    got = np.zeros_like(exp)
    u64p = C.POINTER(C.c_uint64)
    dt = (u64p * len(diags))(*[ptr(d) if d is not None else None for d in diags])
    kt = (u64p * (n // 2))()
    for r, k in keys.items():
        kt[r] = ptr(k)
    ref.L.ref_matvec_bsgs.argtypes = [C.c_void_p, u64p, u64p] + [C.c_int] * 4 + [C.POINTER(u64p)] * 2 + [C.c_int] * 3
    assert ref.L.ref_matvec_bsgs(ref.h, ptr(got), ptr(x), nq, n1, n2, blocks, dt, kt, 0, -1, 1) == 0
    assert np.array_equal(got, exp)
