"""GPU parity: every libhx_b200 entry point vs the CPU oracle, bit-exact
(u64-for-u64) on identical seeded inputs, called through the C-ABI.

Sizes: config 1 (N=2^13, 3+1 primes, alpha=1), a reduced-N config-2 shape
(N=2^12, 24+3 primes, alpha=3) for breadth, and the full config-2 shape
(N=2^16, 24+3 primes) for the NTT and the key-switch family.
"""
import numpy as np
import pytest

from configs import config1, config2, config2_fp64_specials
from oracle_bindings import Oracle, galois_elt, gaussian, ternary, uniform_limbs

pytestmark = pytest.mark.gpu

CFGS = {
    "c1": lambda: config1(13),
    "c2s": lambda: config2(12, 24),
    "c2": lambda: config2(16, 24),
    "c2s47": lambda: config2_fp64_specials(12, 24),  # FP64-class special primes
}

_cache = {}


def env(name):
    if name not in _cache:
        import torch  # noqa: F401

        from paper_2512_11135_b200 import Context

        p = CFGS[name]()
        ctx = Context(p["logn"], p["chain"], p["special"], p["alpha"])
        orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
        _cache[name] = (p, ctx, orc)
    return _cache[name]


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host(t):
    import torch

    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def empty(*shape):
    import torch

    return torch.empty(shape, dtype=torch.int64, device="cuda")


def keyset(p, orc, rng, s_full, sprime_full):
    nq, K = len(p["chain"]), len(p["special"])
    dn = orc.dnum(nq)
    a = uniform_limbs(rng, p["chain"] + p["special"], orc.n, (dn,))
    e = np.stack([gaussian(rng, orc.n) for _ in range(dn)])
    return orc.keygen_ksk(s_full, sprime_full, a, e), a, e


def secret(p, orc, rng):
    nq, K = len(p["chain"]), len(p["special"])
    s = ternary(rng, orc.n)
    return orc.ntt_fwd(orc.from_i64(s, nq, K), nq, K)


# ---------------------------------------------------------------- NTT
@pytest.mark.parametrize("cfg", ["c1", "c2s", "c2"])
def test_ntt_roundtrip_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(1)
    nq, K = len(p["chain"]), len(p["special"])
    batch = 2
    x = uniform_limbs(rng, p["chain"] + p["special"], orc.n, (batch,))
    x[0, 0, :4] = [0, 1, p["chain"][0] - 1, p["chain"][0] - 2]  # edge residues
    d = dev(x)
    ctx.ntt_fwd(d, batch, nq, K)
    got = host(d)
    exp = np.stack([orc.ntt_fwd(x[b], nq, K) for b in range(batch)])
    assert np.array_equal(got, exp)
    ctx.ntt_inv(d, batch, nq, K)
    assert np.array_equal(host(d), x)


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_ntt_extremes(cfg):
    p, ctx, orc = env(cfg)
    nq = len(p["chain"])
    for fill in ("zero", "max"):
        x = np.zeros((nq, orc.n), dtype=np.uint64)
        if fill == "max":
            for i, q in enumerate(p["chain"]):
                x[i] = q - 1
        d = dev(x)
        ctx.ntt_fwd(d, 1, nq, 0)
        assert np.array_equal(host(d), orc.ntt_fwd(x, nq))
        ctx.ntt_inv(d, 1, nq, 0)
        assert np.array_equal(host(d), x)


# ---------------------------------------------------------------- elementwise
@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_elementwise_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(2)
    nq, K = len(p["chain"]), len(p["special"])
    a = uniform_limbs(rng, p["chain"] + p["special"], orc.n)
    b = uniform_limbs(rng, p["chain"] + p["special"], orc.n)
    c = uniform_limbs(rng, p["chain"] + p["special"], orc.n)
    da, db = dev(a), dev(b)
    for name in ("add", "sub", "mul"):
        o = empty(nq + K, orc.n)
        ctx.binop(name, o, da, db, 1, nq, K)
        assert np.array_equal(host(o), orc.binop("hxo_" + name, a, b, nq, K)), name
    o = empty(nq + K, orc.n)
    ctx.neg(o, da, 1, nq, K)
    assert np.array_equal(host(o), orc.neg(a, nq, K))
    dc = dev(c)
    ctx.binop("mul_acc", dc, da, db, 1, nq, K)
    assert np.array_equal(host(dc), orc.mul_acc(c, a, b, nq, K))


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_automorphism_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(3)
    nq, K = len(p["chain"]), len(p["special"])
    a = uniform_limbs(rng, p["chain"] + p["special"], orc.n)
    fa = orc.ntt_fwd(a, nq, K)
    for k in (1, 5, orc.n // 4, orc.n // 2 - 1):
        g = galois_elt(k, orc.n)
        o = empty(nq + K, orc.n)
        ctx.automorphism(o, dev(fa), 1, nq, K, g)
        got = host(o)
        assert np.array_equal(got, orc.automorphism_ntt(fa, nq, K, g))
        # and it is the coefficient-domain automorphism of the reference
        assert np.array_equal(orc.ntt_inv(got, nq, K), orc.automorphism_coeff(a, nq, K, g))


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_rescale_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(4)
    nq = len(p["chain"])
    batch = 3
    x = uniform_limbs(rng, p["chain"], orc.n, (batch,))
    o = empty(batch, nq - 1, orc.n)
    ctx.rescale(o, dev(x), batch, nq)
    got = host(o)
    for b in range(batch):
        assert np.array_equal(got[b], orc.rescale_ntt(x[b], nq))


def test_from_i64_and_reduce():
    p, ctx, orc = env("c2s")
    import torch

    rng = np.random.default_rng(5)
    nq, K = len(p["chain"]), len(p["special"])
    v = rng.integers(-(2**62), 2**62, size=orc.n, dtype=np.int64)
    o = empty(nq + K, orc.n)
    ctx.from_i64(o, torch.from_numpy(v).cuda(), 1, nq, K)
    assert np.array_equal(host(o), orc.from_i64(v, nq, K))
    # reduce_mod_q of a sum of 8 partials (NCCL uint64 sum emulation)
    parts = [uniform_limbs(rng, p["chain"], orc.n) for _ in range(8)]
    tot = np.zeros_like(parts[0])
    for x in parts:
        tot = tot + x  # wraps never: 8 * 2^60 < 2^64
    d = dev(tot)
    ctx.reduce_mod_q(d, 1, nq, 0)
    exp = parts[0]
    for x in parts[1:]:
        exp = orc.binop("hxo_add", exp, x, nq)
    assert np.array_equal(host(d), exp)


# ---------------------------------------------------------------- key switching
@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_modup_inner_moddown_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(6)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    key, _, _ = keyset(p, orc, rng, s_full, orc.automorphism_ntt(s_full, nq, K, galois_elt(3, orc.n)))
    dkey = dev(key)
    for lvl in sorted({nq, max(1, nq - 2), 1}, reverse=True):
        batch = 2
        c1 = uniform_limbs(rng, p["chain"][:lvl], orc.n, (batch,))
        dn = orc.dnum(lvl)
        D = empty(batch, dn, lvl + K, orc.n)
        ctx.modup(D, dev(c1), batch, lvl)
        Dg = host(D)
        for b in range(batch):
            assert np.array_equal(Dg[b], orc.modup(c1[b], lvl)), f"modup lvl={lvl}"
        g = galois_elt(7, orc.n)
        U = empty(batch, 2, lvl + K, orc.n)
        ctx.ks_inner(U, D, dkey, batch, lvl, g)
        Ug = host(U)
        for b in range(batch):
            assert np.array_equal(Ug[b], orc.ks_inner(Dg[b], key, lvl, g)), f"inner lvl={lvl}"
        V = empty(batch, 2, lvl, orc.n)
        ctx.moddown(V, U, 2 * batch, lvl)
        Vg = host(V)
        for b in range(batch):
            assert np.array_equal(Vg[b], orc.moddown_ntt(Ug[b], lvl, 2)), f"moddown lvl={lvl}"


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c2", "c2s47"])
def test_rotate_parity_and_decrypt(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(7)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    k = 3
    g = galois_elt(k, orc.n)
    key, _, _ = keyset(p, orc, rng, s_full, orc.automorphism_ntt(s_full, nq, K, g))
    batch = 2 if cfg != "c2" else 1
    mcoef = rng.integers(-(2**20), 2**20, size=(batch, orc.n)).astype(np.int64)
    cts = []
    for b in range(batch):
        m_ntt = orc.ntt_fwd(orc.from_i64(mcoef[b], nq), nq)
        cts.append(orc.encrypt_sk(m_ntt, s_full, uniform_limbs(rng, p["chain"], orc.n), gaussian(rng, orc.n), nq))
    ct = np.stack(cts)
    out = empty(batch, 2, nq, orc.n)
    ctx.rotate(out, dev(ct), ctx.rotation_key(dev(key), g), batch, nq, g)
    got = host(out)
    for b in range(batch):
        exp = orc.rotate(ct[b], key, nq, g)
        assert np.array_equal(got[b], exp)
        # decrypts to tau_g(m) up to small key-switching noise
        dec = orc.ntt_inv(orc.decrypt(got[b], s_full, nq), nq)
        ref = orc.automorphism_coeff(orc.from_i64(mcoef[b], nq), nq, 0, g)
        q0 = p["chain"][0]
        diff = (dec[0].astype(object) - ref[0].astype(object)) % q0
        diff = np.where(diff > q0 // 2, diff - q0, diff)
        assert np.abs(diff).max() < 2**16


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c2s47"])
def test_keyswitch_and_hoisted_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(8)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    ks = [1, 2, 5, 16]
    gs = [galois_elt(k, orc.n) for k in ks]
    keys = [keyset(p, orc, rng, s_full, orc.automorphism_ntt(s_full, nq, K, g))[0] for g in gs]
    ct = uniform_limbs(rng, p["chain"], orc.n, (2,))
    # plain key switch of c1
    out = empty(2, nq, orc.n)
    ctx.keyswitch(out, dev(ct[1]), dev(keys[0]), 1, nq)
    assert np.array_equal(host(out), orc.keyswitch(ct[1], keys[0], nq))
    # hoisted batch
    dkeys = [ctx.rotation_key(dev(k), g) for k, g in zip(keys, gs)]
    outh = empty(1, len(gs), 2, nq, orc.n)
    ctx.rotate_hoisted(outh, dev(ct), dkeys, gs, 1, nq)
    exp = orc.rotate_hoisted(ct, keys, gs, nq)
    assert np.array_equal(host(outh)[0], exp)
    # hoisted == independent rotations (same convention)
    for r, g in enumerate(gs):
        assert np.array_equal(exp[r], orc.rotate(ct, keys[r], nq, g))


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c2s47", "c2"])
def test_rotate_multi_parity(cfg):
    """hx_rotate_multi: per-element keys / galois elements, one batched ModUp
    (the fused ROW + inner-product kernel with a key per element; "c2" at
    the N = 2^16 tile shape)"""
    import ctypes as C

    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(14)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    ks = [3, 8, 40]
    gs = [galois_elt(k, orc.n) for k in ks]
    keys = [keyset(p, orc, rng, s_full, orc.automorphism_ntt(s_full, nq, K, g))[0] for g in gs]
    dkeys = [ctx.rotation_key(dev(k), g) for k, g in zip(keys, gs)]
    cts = uniform_limbs(rng, p["chain"], orc.n, (3, 2))
    out = empty(3, 2, nq, orc.n)
    kp = (C.c_void_p * 3)(*[k.data_ptr() for k in dkeys])
    ga = (C.c_uint64 * 3)(*gs)
    ctx.L.hx_rotate_multi.argtypes = [C.c_void_p] * 4 + [C.POINTER(C.c_uint64), C.c_int, C.c_int, C.c_void_p]
    assert ctx.L.hx_rotate_multi(ctx.h, out.data_ptr(), dev(cts).data_ptr(), kp, ga, 3, nq, None) == 0
    got = host(out)
    for b in range(3):
        assert np.array_equal(got[b], orc.rotate(cts[b], keys[b], nq, gs[b])), b


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c2s47"])
def test_tensor_and_mul_relin_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(9)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    s2 = orc.binop("hxo_mul", s_full, s_full, nq, K)
    rlk, _, _ = keyset(p, orc, rng, s_full, s2)
    batch = 2
    a = uniform_limbs(rng, p["chain"], orc.n, (batch, 2))
    b = uniform_limbs(rng, p["chain"], orc.n, (batch, 2))
    o3 = empty(batch, 3, nq, orc.n)
    ctx.tensor(o3, dev(a), dev(b), batch, nq)
    got3 = host(o3)
    o = empty(batch, 2, nq, orc.n)
    ctx.mul_relin(o, dev(a), dev(b), dev(rlk), batch, nq)
    got = host(o)
    for i in range(batch):
        assert np.array_equal(got3[i], orc.tensor(a[i], b[i], nq))
        assert np.array_equal(got[i], orc.mul_relin(a[i], b[i], rlk, nq))


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_bsgs_mac_parity(cfg):
    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(10)
    nq = len(p["chain"])
    for n1, n2 in ((8, 8), (4, 2), (3, 5), (32, 2)):
        lvl = nq
        baby = uniform_limbs(rng, p["chain"][:lvl], orc.n, (n1, 2))
        diags = uniform_limbs(rng, p["chain"][:lvl], orc.n, (n2 * n1,))
        o = empty(n2, 2, lvl, orc.n)
        ctx.bsgs_mac(o, dev(baby), dev(diags), lvl, n1, n2, lvl)
        assert np.array_equal(host(o), orc.bsgs_mac(baby, diags, n1, n2, lvl)), (n1, n2)


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_keygen_encrypt_decrypt_parity(cfg):
    import torch

    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(11)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    sp = orc.automorphism_ntt(s_full, nq, K, galois_elt(9, orc.n))
    dn = orc.dnum(nq)
    a = uniform_limbs(rng, p["chain"] + p["special"], orc.n, (dn,))
    e = np.stack([gaussian(rng, orc.n) for _ in range(dn)])
    key = empty(ctx.key_words())
    ctx.keygen_ksk(key, dev(s_full), dev(sp), dev(a), torch.from_numpy(e).cuda())
    assert np.array_equal(host(key).reshape(dn, 2, nq + K, orc.n), orc.keygen_ksk(s_full, sp, a, e))
    m = uniform_limbs(rng, p["chain"], orc.n)
    ca = uniform_limbs(rng, p["chain"], orc.n)
    ee = gaussian(rng, orc.n)
    ct = empty(2, nq, orc.n)
    ctx.encrypt_sk(ct, dev(m), dev(s_full), dev(ca), torch.from_numpy(ee).cuda(), nq)
    exp = orc.encrypt_sk(m, s_full, ca, ee, nq)
    assert np.array_equal(host(ct), exp)
    mo = empty(1, nq, orc.n)
    ctx.decrypt(mo, ct, dev(s_full), 1, nq)
    assert np.array_equal(host(mo)[0], orc.decrypt(exp, s_full, nq))


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_keygen_rotation_layout(cfg):
    """hx_keygen_rotation == hx_ksk_to_rotation_layout(standard keygen of tau_g(s))."""
    import torch

    p, ctx, orc = env(cfg)
    rng = np.random.default_rng(13)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    g = galois_elt(11, orc.n)
    dn = orc.dnum(nq)
    a = uniform_limbs(rng, p["chain"] + p["special"], orc.n, (dn,))
    e = np.stack([gaussian(rng, orc.n) for _ in range(dn)])
    std = orc.keygen_ksk(s_full, orc.automorphism_ntt(s_full, nq, K, g), a, e)
    key = empty(ctx.key_words())
    ctx.keygen_rotation(key, dev(s_full), g, dev(a), torch.from_numpy(e).cuda())
    assert np.array_equal(host(key), host(ctx.rotation_key(dev(std), g)).reshape(-1))
    # and the rotation layout is tau_{g^-1} of the standard layout, limb-wise
    ginv = pow(g, -1, 2 * orc.n)
    exp = orc.automorphism_ntt(std.reshape(dn * 2 * (nq + K), orc.n), dn * 2 * (nq + K), 0, ginv)
    assert np.array_equal(host(key).reshape(-1, orc.n), exp)


def test_host_entry_points():
    """hx_rotate_host / hx_mul_relin_host (host buffers in, host buffers out)."""
    import torch

    p, ctx, orc = env("c2s")
    rng = np.random.default_rng(12)
    nq, K = len(p["chain"]), len(p["special"])
    s_full = secret(p, orc, rng)
    g = galois_elt(1, orc.n)
    key, _, _ = keyset(p, orc, rng, s_full, orc.automorphism_ntt(s_full, nq, K, g))
    ct = uniform_limbs(rng, p["chain"], orc.n, (2, 2))
    out = np.zeros_like(ct)
    ctx.rotate_host(out.ctypes.data, ct.ctypes.data, ctx.rotation_key(dev(key), g), 2, nq, g)
    for b in range(2):
        assert np.array_equal(out[b], orc.rotate(ct[b], key, nq, g))
    s2 = orc.binop("hxo_mul", s_full, s_full, nq, K)
    rlk, _, _ = keyset(p, orc, rng, s_full, s2)
    ct2 = uniform_limbs(rng, p["chain"], orc.n, (2, 2))
    ctx.mul_relin_host(out.ctypes.data, ct.ctypes.data, ct2.ctypes.data, dev(rlk), 2, nq)
    for b in range(2):
        assert np.array_equal(out[b], orc.mul_relin(ct[b], ct2[b], rlk, nq))
    del torch


def test_errors_are_loud():
    from paper_2512_11135_b200 import HxError

    p, ctx, orc = env("c1")
    with pytest.raises(HxError):
        ctx.rescale(empty(1, orc.n), empty(1, orc.n), 1, 1)  # no limb to drop
    with pytest.raises(HxError):
        ctx.automorphism(empty(1, orc.n), empty(1, orc.n), 1, 1, 0, 4)  # even galois element


def test_device_samplers():
    """key-material samplers: uniform residues below each limb's prime with
    uniform-looking moments, centred binomial errors in [-21, 21] with the
    k = 21 variance; distinct seeds give distinct streams."""
    p, ctx, orc = env("c2s")
    nq, K, N = len(p["chain"]), len(p["special"]), 1 << p["logn"]
    out = empty(2, nq + K, N)
    ctx.sample_uniform(out, nq, K, 2, 1234)
    u = host(out).view(np.uint64)
    primes = np.array(p["chain"] + p["special"], dtype=np.uint64)
    assert (u < primes[None, :, None]).all()
    frac = u.astype(np.float64) / primes[None, :, None].astype(np.float64)
    assert abs(frac.mean() - 0.5) < 0.01 and abs(frac.var() - 1 / 12) < 0.005
    e = empty(4 * N)
    ctx.sample_cbd(e, 4 * N, 99)
    ev = host(e).view(np.int64)
    assert ev.min() >= -21 and ev.max() <= 21
    assert abs(ev.mean()) < 0.1 and abs(ev.var() - 10.5) < 0.5
    out2 = empty(2, nq + K, N)
    ctx.sample_uniform(out2, nq, K, 2, 1235)
    assert not np.array_equal(host(out2), host(out))


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_compressed_keys(cfg):
    """SURVEY 8(f)-2 seeded key compression: a compressed key (b halves only,
    the uniform halves regenerated from the seed inside the inner product)
    expands to exactly the full key made from hx_sample_uniform(seed), and a
    rotation / key switch with it gives the same words as with the full key."""
    p, ctx, orc = env(cfg)
    import torch

    from paper_2512_11135_b200.hx import lib

    nq, K, N = len(p["chain"]), len(p["special"]), 1 << p["logn"]
    rng = np.random.default_rng(91)
    s_full = dev(secret(p, orc, rng))
    dn = orc.dnum(len(p["chain"]))
    e = dev(np.ascontiguousarray(np.stack([gaussian(rng, N) for _ in range(dn)]).astype(np.int64)))
    L = lib()
    import ctypes as C

    L.hx_ckey_words.restype = C.c_size_t
    L.hx_ckey_words.argtypes = [C.c_void_p]
    for fn in ("hx_keygen_rotation_c",):
        getattr(L, fn).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
    L.hx_key_expand.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.hx_key_release.argtypes = [C.c_void_p, C.c_void_p]
    seed, g = 0x1234ABCD, galois_elt(3, N)
    ck = torch.empty(int(L.hx_ckey_words(ctx.h)), dtype=torch.int64, device="cuda")
    assert L.hx_keygen_rotation_c(ctx.h, ck.data_ptr(), s_full.data_ptr(), g, seed, e.data_ptr(), None) == 0
    full_c = torch.empty(ctx.key_words(), dtype=torch.int64, device="cuda")
    assert L.hx_key_expand(ctx.h, full_c.data_ptr(), ck.data_ptr(), None) == 0
    # the same key from explicit uniform words of the same seed
    a = empty(dn, nq + K, N)
    ctx.sample_uniform(a, nq, K, dn, seed)
    full = torch.empty(ctx.key_words(), dtype=torch.int64, device="cuda")
    ctx.keygen_rotation(full, s_full, g, a, e)
    assert np.array_equal(host(full_c), host(full))
    # rotations with the compressed and the full key agree word for word
    ct = dev(uniform_limbs(rng, p["chain"], N, (2, 2)))
    o1, o2 = empty(2, 2, nq, N), empty(2, 2, nq, N)
    ctx.rotate(o1, ct, ck, 2, nq, g)
    ctx.rotate(o2, ct, full, 2, nq, g)
    assert np.array_equal(host(o1), host(o2))
    assert L.hx_key_release(ctx.h, ck.data_ptr()) == 0


def test_ntt_cluster_variant_parity():
    """The opt-in single-pass cluster NTT (HX_NTT_CLUSTER=1, read once per
    process, hence the subprocess) gives the same words as the oracle at
    N = 2^16: forward, inverse, and the out-of-place inverse of ModUp inside a
    key switch (via the full rotate parity test)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env_ = dict(os.environ, HX_NTT_CLUSTER="1")
    f = os.path.join(here, "test_gpu_parity.py")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        f + "::test_ntt_roundtrip_parity[c2]", f + "::test_rotate_parity_and_decrypt[c2]"],
                       env=env_, capture_output=True, text=True, cwd=here, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout and "2 passed" in r.stdout, r.stdout[-2000:]
