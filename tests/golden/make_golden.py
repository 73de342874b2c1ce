"""Generate tests/golden/*.npz from the REFERENCE's own compiled code
(oracle/_ref/libhelix_ref.so = /root/reference/proj/src/*.cpp with the
modmath.hpp:30 Barrett fix, see oracle/Makefile).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
The fixtures pin the C oracle (tests/test_oracle.py) and travel with the repo;
nothing at test time reads /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_bindings import Ref, find_ntt_primes, f64p, galois_elt, gaussian, ptr, ternary, uniform_limbs  # noqa: E402

LOGN = 10
N = 1 << LOGN


def main():
    rng = np.random.default_rng(20251211)
    # config-1 prime shapes (= 1 mod 2^14, hence usable at N = 2^10)
    chain = find_ntt_primes(1 << 39, 3, 1 << 14)
    special = find_ntt_primes(1 << 49, 1, 1 << 14)
    primes = chain + special
    r = Ref(LOGN, chain, special, 1, 40)
    L = r.L
    out = {"logn": np.array(LOGN), "chain": np.array(chain, dtype=np.uint64),
           "special": np.array(special, dtype=np.uint64)}
    out["psi"] = np.array([L.ref_psi(r.h, i) for i in range(4)], dtype=np.uint64)
    # NttTables::forward / inverse (ntt.cpp:57-96)
    x = uniform_limbs(rng, primes, N)
    out["ntt_in"] = x
    out["ntt_fwd"] = np.stack([r.ntt_fwd(i, x[i]) for i in range(4)])
    out["ntt_inv"] = np.stack([r.ntt_inv(i, x[i]) for i in range(4)])
    # LatticeContext::automorphism (rns_poly.cpp:124-142), coefficient domain
    a = uniform_limbs(rng, chain, N)
    out["auto_in"] = a
    out["auto_g"] = np.array([galois_elt(k, N) for k in (1, 3, 100)], dtype=np.uint64)
    res = []
    for g in out["auto_g"]:
        o = np.zeros_like(a)
        assert L.ref_lc_automorphism(r.h, ptr(a), ptr(o), 3, 0, int(g)) == 0
        res.append(o)
    out["auto_out"] = np.stack(res)
    # rescale_drop_last (rns_poly.cpp:144-162)
    o = np.zeros((2, N), dtype=np.uint64)
    assert L.ref_lc_rescale(r.h, ptr(a), ptr(o), 3) == 0
    out["rescale_out"] = o
    # moddown_special (rns_poly.cpp:164-180)
    ax = uniform_limbs(rng, primes, N)
    out["moddown_in"] = ax
    o = np.zeros((3, N), dtype=np.uint64)
    assert L.ref_lc_moddown(r.h, ptr(ax), ptr(o), 3) == 0
    out["moddown_out"] = o
    # mul_acc (rns_poly.cpp:102-110) and ring_mul (:112-122)
    b = uniform_limbs(rng, chain, N)
    acc = uniform_limbs(rng, chain, N)
    out["mac_a"], out["mac_b"], out["mac_acc"] = a, b, acc.copy()
    assert L.ref_lc_mul_acc(r.h, ptr(a), ptr(b), ptr(acc), 3) == 0
    out["mac_out"] = acc
    o = np.zeros((3, N), dtype=np.uint64)
    assert L.ref_lc_ring_mul(r.h, ptr(a), ptr(b), ptr(o), 3) == 0
    out["ring_mul_out"] = o
    # CkksEncoder::encode / decode (encoder.cpp:97-159)
    m = rng.uniform(-1, 1, 64)
    out["enc_m"] = m
    o = np.zeros((3, N), dtype=np.uint64)
    assert L.ref_encode(r.h, ptr(m, f64p), len(m), 2, float(2**40), ptr(o)) == 0
    out["enc_out"] = o
    dec = np.zeros(N // 2)
    assert L.ref_decode(r.h, ptr(o), 3, float(2**40), ptr(dec, f64p)) == 0
    out["dec_out"] = dec
    # key switch composed over the reference primitives (ref_shim.cpp)
    from oracle_bindings import Oracle

    orc = Oracle(LOGN, chain, special, 1)  # only to build a key from (s, a, e)
    s_full = orc.ntt_fwd(orc.from_i64(ternary(rng, N), 3, 1), 3, 1)
    g = galois_elt(5, N)
    sp = orc.automorphism_ntt(s_full, 3, 1, g)
    ka = uniform_limbs(rng, primes, N, (3,))
    ke = np.stack([gaussian(rng, N) for _ in range(3)])
    key = orc.keygen_ksk(s_full, sp, ka, ke)
    ct = uniform_limbs(rng, chain, N, (2,))
    o = np.zeros_like(ct)
    assert L.ref_rotate(r.h, ptr(ct), ptr(key), ptr(o), 3, g) == 0
    out.update(ks_key=key, ks_ct=ct, ks_g=np.array(g), ks_out=o)
    np.savez_compressed(os.path.join(HERE, "ref_n1024.npz"), **out)
    print("wrote", os.path.join(HERE, "ref_n1024.npz"))


if __name__ == "__main__":
    main()
