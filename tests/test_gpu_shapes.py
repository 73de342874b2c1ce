"""GPU parity at the BENCHMARKED launch shapes (VERDICT r1 "next round" 1).

Every call here is the exact call bench.py times (or its grid-shape twin),
compared word for word with the CPU oracle on sampled outputs:

  * hx_rotate at N = 2^16, 24 + 3 primes (60-bit specials), batch 256 -- the
    headline step (modup_col with tsplit == 1, ks_row_inner over the whole
    batch); ciphertexts 0, 1, the middle ones and the last ones vs hxo_rotate;
  * hx_mul_relin at N = 2^16, batch 32;
  * hx_rotate_hoisted at N = 2^16 with R = 32 DISTINCT rotation keys;
  * hx_modup / hx_ks_inner / hx_moddown at N = 2^16, batch 32 (ks_inner
    element slices = 2; the batch-64 shape at N = 2^12 below reaches 4);
  * hx_bsgs_mac at N = 2^16, n1 = n2 = 32, 24 limbs (the FFN W1 block):
    limbs of both kernel classes (60-bit integer, 40-bit FP64) vs the oracle;
  * batch >= 64 at N = 2^12 / 2^13 through hx_rotate, hx_rotate_multi and
    hx_rotate_grouped, all outputs vs the oracle (tsplit == 1, slices > 1).

Inputs are uniform residues sampled on the device (hx_sample_uniform) and
keys generated on the device in the STANDARD layout (hx_keygen_ksk) -- the
oracle receives the same words; the GPU rotation calls take the rotation
layout made from them (hx_ksk_to_rotation_layout).  Keygen itself is checked
against the oracle at smaller N in test_gpu_parity.py.
"""
import numpy as np
import pytest

from configs import config1, config2
from oracle_bindings import Oracle, galois_elt

pytestmark = pytest.mark.gpu

_cache = {}


def env(name):
    if name not in _cache:
        import torch  # noqa: F401

        from paper_2512_11135_b200 import Context

        p = {"c2": lambda: config2(16, 24), "c2s": lambda: config2(12, 24), "c1": lambda: config1(13)}[name]()
        ctx = Context(p["logn"], p["chain"], p["special"], p["alpha"])
        orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
        _cache[name] = (p, ctx, orc)
    return _cache[name]


def host(t):
    import torch

    torch.cuda.synchronize()
    return np.ascontiguousarray(t.cpu().numpy().view(np.uint64))


def empty(*shape):
    import torch

    return torch.empty(shape, dtype=torch.int64, device="cuda")


def dev_uniform(ctx, n_c, n_s, copies, seed):
    t = empty(copies, n_c + n_s, ctx.n)
    ctx.sample_uniform(t, n_c, n_s, copies, seed)
    return t


def dev_secret(ctx, nq, K, seed):
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    s = torch.randint(-1, 2, (ctx.n,), generator=g, device="cuda", dtype=torch.int64)
    s_full = empty(nq + K, ctx.n)
    ctx.from_i64(s_full, s, 1, nq, K)
    ctx.ntt_fwd(s_full, 1, nq, K)
    return s_full


def dev_key(ctx, s_full, nq, K, galois, seed):
    """standard-layout switching key (device) for s' = tau_g(s), or s^2 if galois == 0"""
    sp = empty(nq + K, ctx.n)
    if galois == 0:
        ctx.binop("mul", sp, s_full, s_full, 1, nq, K)
    else:
        ctx.automorphism(sp, s_full, 1, nq, K, galois)
    dn = ctx.dnum(nq)
    a = dev_uniform(ctx, nq, K, dn, seed)
    e = empty(dn * ctx.n)
    ctx.sample_cbd(e, dn * ctx.n, seed + 1)
    key = empty(ctx.key_words())
    ctx.keygen_ksk(key, s_full, sp, a, e)
    return key


def key_host(ctx, orc, key, nq_full, K):
    return host(key).reshape(orc.dnum(nq_full), 2, nq_full + K, ctx.n)


def sample_idx(batch):
    return sorted({0, 1, batch // 2 - 1, batch // 2, batch - 2, batch - 1})


# ------------------------------------------------------------ the headline step
def test_headline_rotate_batch256_n16():
    """bench.py's timed call: hx_rotate over 256 ciphertexts at N = 2^16."""
    p, ctx, orc = env("c2")
    nq, K, B = 24, 3, 256
    g = galois_elt(1, ctx.n)
    s = dev_secret(ctx, nq, K, 11)
    key = dev_key(ctx, s, nq, K, g, 1000)
    rkey = ctx.rotation_key(key, g)
    cts = dev_uniform(ctx, nq, 0, 2 * B, 2024).view(B, 2, nq, ctx.n)
    out = empty(B, 2, nq, ctx.n)
    ctx.rotate(out, cts, rkey, B, nq, g)
    kh = key_host(ctx, orc, key, nq, K)
    for b in sample_idx(B):
        exp = orc.rotate(host(cts[b]), kh, nq, g)
        assert np.array_equal(host(out[b]), exp), f"ciphertext {b} of 256"


def test_headline_rotate_lower_level_batch64_n16():
    """the same key over a lower level (16 limbs: dnum 6 of the key's 8 digits)"""
    p, ctx, orc = env("c2")
    nq, K, B = 16, 3, 64
    g = galois_elt(5, ctx.n)
    s = dev_secret(ctx, 24, K, 12)
    key = dev_key(ctx, s, 24, K, g, 1100)
    rkey = ctx.rotation_key(key, g)
    cts = dev_uniform(ctx, nq, 0, 2 * B, 77).view(B, 2, nq, ctx.n)
    out = empty(B, 2, nq, ctx.n)
    ctx.rotate(out, cts, rkey, B, nq, g)
    kh = key_host(ctx, orc, key, 24, K)
    for b in (0, B - 1):
        assert np.array_equal(host(out[b]), orc.rotate(host(cts[b]), kh, nq, g)), b


def test_mul_relin_batch32_n16():
    p, ctx, orc = env("c2")
    nq, K, B = 24, 3, 32
    s = dev_secret(ctx, nq, K, 13)
    rlk = dev_key(ctx, s, nq, K, 0, 1200)
    a = dev_uniform(ctx, nq, 0, 2 * B, 5).view(B, 2, nq, ctx.n)
    b = dev_uniform(ctx, nq, 0, 2 * B, 6).view(B, 2, nq, ctx.n)
    out = empty(B, 2, nq, ctx.n)
    ctx.mul_relin(out, a, b, rlk, B, nq)
    kh = key_host(ctx, orc, rlk, nq, K)
    for i in (0, 15, 31):
        assert np.array_equal(host(out[i]), orc.mul_relin(host(a[i]), host(b[i]), kh, nq)), i


def test_hoisted32_distinct_keys_n16():
    """bench.py's hoisted extra with 32 DISTINCT keys (rotations by 1..32)"""
    import torch

    p, ctx, orc = env("c2")
    nq, K, B, R = 24, 3, 8, 32
    s = dev_secret(ctx, nq, K, 14)
    gs = [galois_elt(k, ctx.n) for k in range(1, R + 1)]
    std = [dev_key(ctx, s, nq, K, g, 2000 + 7 * r) for r, g in enumerate(gs)]
    rkeys = [ctx.rotation_key(k, g) for k, g in zip(std, gs)]
    cts = dev_uniform(ctx, nq, 0, 2 * B, 31).view(B, 2, nq, ctx.n)
    out = empty(B, R, 2, nq, ctx.n)
    ctx.rotate_hoisted(out, cts, rkeys, gs, B, nq)
    torch.cuda.synchronize()
    del rkeys
    kh = [key_host(ctx, orc, k, nq, K) for k in std]
    del std
    for b in (0, B - 1):
        exp = orc.rotate_hoisted(host(cts[b]), kh, gs, nq)
        got = host(out[b])
        for r in range(R):
            assert np.array_equal(got[r], exp[r]), (b, r)


def test_modup_inner_moddown_batch32_n16():
    p, ctx, orc = env("c2")
    nq, K, B = 24, 3, 32
    dn = ctx.dnum(nq)
    s = dev_secret(ctx, nq, K, 15)
    g = galois_elt(9, ctx.n)
    key = dev_key(ctx, s, nq, K, g, 1300)
    c1 = dev_uniform(ctx, nq, 0, B, 8).view(B, nq, ctx.n)
    D = empty(B, dn, nq + K, ctx.n)
    ctx.modup(D, c1, B, nq)
    U = empty(B, 2, nq + K, ctx.n)
    ctx.ks_inner(U, D, key, B, nq, g)
    V = empty(B, 2, nq, ctx.n)
    ctx.moddown(V, U, 2 * B, nq)
    kh = key_host(ctx, orc, key, nq, K)
    for b in (0, B - 1):
        Db = orc.modup(host(c1[b]), nq)
        assert np.array_equal(host(D[b]), Db), f"modup {b}"
        Ub = orc.ks_inner(Db, kh, nq, g)
        assert np.array_equal(host(U[b]), Ub), f"inner {b}"
        assert np.array_equal(host(V[b]), orc.moddown_ntt(Ub, nq, 2)), f"moddown {b}"


def test_bsgs_mac_w1_block_n16():
    """n1 = n2 = 32 over 24 limbs at N = 2^16 (1024 diagonals, 12.9 GB): the
    MAC of one FFN W1 block; limb 0 (60-bit, 128-bit integer kernel) and
    40-bit limbs (FP64 kernel) vs a one-prime oracle per limb."""
    import torch

    p, ctx, orc = env("c2")
    nq, n1, n2 = 24, 32, 32
    baby = dev_uniform(ctx, nq, 0, n1 * 2, 41).view(n1, 2, nq, ctx.n)
    diags = dev_uniform(ctx, nq, 0, n1 * n2, 42).view(n1 * n2, nq, ctx.n)
    inner = empty(n2, 2, nq, ctx.n)
    ctx.bsgs_mac(inner, baby, diags, nq, n1, n2, nq)
    torch.cuda.synchronize()
    for k in (0, 1, 12, 23):
        o1 = Oracle(p["logn"], [p["chain"][k]], [], 1)
        bk = host(baby[:, :, k, :].contiguous()).reshape(n1, 2, 1, ctx.n)
        dk = host(diags[:, k, :].contiguous()).reshape(n1 * n2, 1, ctx.n)
        exp = o1.bsgs_mac(bk, dk, n1, n2, 1)
        got = host(inner[:, :, k, :].contiguous()).reshape(n2, 2, 1, ctx.n)
        assert np.array_equal(got, exp), f"limb {k}"


# ------------------------------------------------------------ large batches at small N
@pytest.mark.parametrize("name,B", [("c2s", 64), ("c2s", 96), ("c1", 64)])
def test_large_batch_rotations_all_outputs(name, B):
    """batch >= 64 takes modup_col's tsplit == 1 grid and ks_inner's
    multi-slice grid; hx_rotate, hx_rotate_multi (one key per element) and
    hx_rotate_grouped (E = B / 4 per key) vs the oracle on EVERY output."""
    p, ctx, orc = env(name)
    nq, K = len(p["chain"]), len(p["special"])
    s = dev_secret(ctx, nq, K, 16)
    ks = [1, 3, 7, 100]
    gs = [galois_elt(k, ctx.n) for k in ks]
    std = [dev_key(ctx, s, nq, K, g, 3000 + r) for r, g in enumerate(gs)]
    rkeys = [ctx.rotation_key(k, g) for k, g in zip(std, gs)]
    kh = [key_host(ctx, orc, k, nq, K) for k in std]
    cts = dev_uniform(ctx, nq, 0, 2 * B, 55 + B).view(B, 2, nq, ctx.n)
    ch = host(cts)
    out = empty(B, 2, nq, ctx.n)
    ctx.rotate(out, cts, rkeys[0], B, nq, gs[0])
    got = host(out)
    exp0 = [orc.rotate(ch[b], kh[0], nq, gs[0]) for b in range(B)]
    for b in range(B):
        assert np.array_equal(got[b], exp0[b]), f"hx_rotate {b}"
    # per-element keys: element b uses key b % 4
    ctx.rotate_multi(out, cts, [rkeys[b % 4] for b in range(B)], [gs[b % 4] for b in range(B)], nq)
    got = host(out)
    for b in range(B):
        r = b % 4
        exp = exp0[b] if r == 0 else orc.rotate(ch[b], kh[r], nq, gs[r])
        assert np.array_equal(got[b], exp), f"hx_rotate_multi {b}"
    # grouped: group r = ciphertexts r*E .. r*E+E-1 with key r
    E = B // 4
    ctx.rotate_grouped(out, cts, rkeys, gs, E, nq)
    got = host(out)
    for b in range(B):
        r = b // E
        exp = exp0[b] if r == 0 else orc.rotate(ch[b], kh[r], nq, gs[r])
        assert np.array_equal(got[b], exp), f"hx_rotate_grouped {b}"


@pytest.mark.parametrize("name,B", [("c2s", 64)])
def test_large_batch_ks_inner_slices(name, B):
    """hx_ks_inner with E = 64 elements over one key (8 element slices)"""
    p, ctx, orc = env(name)
    nq, K = len(p["chain"]), len(p["special"])
    dn = ctx.dnum(nq)
    s = dev_secret(ctx, nq, K, 17)
    g = galois_elt(3, ctx.n)
    key = dev_key(ctx, s, nq, K, g, 4000)
    c1 = dev_uniform(ctx, nq, 0, B, 9).view(B, nq, ctx.n)
    D = empty(B, dn, nq + K, ctx.n)
    ctx.modup(D, c1, B, nq)
    U = empty(B, 2, nq + K, ctx.n)
    ctx.ks_inner(U, D, key, B, nq, g)
    Dh, Uh = host(D), host(U)
    kh = key_host(ctx, orc, key, nq, K)
    c1h = host(c1)
    for b in range(B):
        assert np.array_equal(Dh[b], orc.modup(c1h[b], nq)), f"modup {b}"
        assert np.array_equal(Uh[b], orc.ks_inner(Dh[b], kh, nq, g)), f"inner {b}"


def test_bsgs_mac_sparse_pruned_w1_block_n16():
    """the index-list MAC of a 90 %-pruned W1 block (n1 = n2 = 32, 24 limbs,
    N = 2^16, 2 tokens) vs the oracle MAC with the dead diagonals zeroed"""
    import torch

    p, ctx, orc = env("c2")
    nq, n1, n2, T = 24, 32, 32, 2
    rng = np.random.default_rng(43)
    live = sorted(rng.choice(n1 * n2, 102, replace=False).tolist())
    baby = dev_uniform(ctx, nq, 0, T * n1 * 2, 44).view(T, n1, 2, nq, ctx.n)
    diags = dev_uniform(ctx, nq, 0, len(live), 45).view(len(live), nq, ctx.n)
    gptr, ks, ptrs = [0], [], []
    for j in range(n2):
        for e, idx in enumerate(live):
            if idx // n1 == j:
                ks.append(idx % n1)
                ptrs.append(diags[e].data_ptr())
        gptr.append(len(ks))
    ctw = 2 * nq * ctx.n
    inner = torch.zeros((T, n2, 2, nq, ctx.n), dtype=torch.int64, device="cuda")
    ctx.bsgs_mac_sparse(inner, ctw, baby, gptr, ks, ptrs, n1, n2, nq, tokens=T,
                        inner_tstride=n2 * ctw, baby_tstride=n1 * ctw)
    torch.cuda.synchronize()
    for k in (0, 5):
        o1 = Oracle(p["logn"], [p["chain"][k]], [], 1)
        dense = np.zeros((n1 * n2, 1, ctx.n), dtype=np.uint64)
        dh = host(diags[:, k, :].contiguous())
        for e, idx in enumerate(live):
            dense[idx, 0] = dh[e]
        for t in range(T):
            bk = host(baby[t, :, :, k, :].contiguous()).reshape(n1, 2, 1, ctx.n)
            exp = o1.bsgs_mac(bk, dense, n1, n2, 1)
            got = host(inner[t, :, :, k, :].contiguous()).reshape(n2, 2, 1, ctx.n)
            assert np.array_equal(got, exp), (k, t)
