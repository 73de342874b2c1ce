"""Edge cases of the device C-ABI (include/hx_b200.h): empty batches are
no-ops, malformed shapes and Galois elements fail with HX_ERR_INVALID and a
message (never a silent result or a CUDA launch error), ragged matrices
(last row block partially filled, rectangular wider than tall) and the
largest supported BSGS shape at N = 2^12 stay exact, and rotations by
multiples of the slot count need no key (reference_backend.cpp:106)."""
import numpy as np
import pytest

from configs import config2

pytestmark = pytest.mark.gpu


def _ctx():
    import torch  # noqa: F401

    from paper_2512_11135_b200 import Context

    p = config2(12, 24)
    return p, Context(p["logn"], p["chain"], p["special"], p["alpha"])


def _empty(*shape):
    import torch

    return torch.zeros(shape, dtype=torch.int64, device="cuda")


def test_empty_batches_are_noops():
    p, ctx = _ctx()
    nq, N = len(p["chain"]), 1 << p["logn"]
    x = _empty(1, 2, nq, N)
    y = _empty(1, 2, nq, N)
    key = _empty(ctx.dnum(nq), 2, nq + len(p["special"]), N)
    ctx.ntt_fwd(x, 0, nq)
    ctx.ntt_inv(x, 0, nq)
    ctx.binop("add", x, x, x, 0, nq)
    ctx.reduce_mod_q(x, 0, nq)
    ctx.rotate(y, x, key, 0, nq, 5)
    ctx.mul_relin(y, x, x, key, 0, nq)
    import torch

    torch.cuda.synchronize()
    assert int(x.abs().sum()) == 0 and int(y.abs().sum()) == 0


def test_invalid_arguments_fail_loudly():
    from paper_2512_11135_b200.hx import HxError

    p, ctx = _ctx()
    nq, N = len(p["chain"]), 1 << p["logn"]
    x = _empty(1, 2, nq, N)
    y = _empty(1, 2, nq, N)
    key = _empty(ctx.dnum(nq), 2, nq + len(p["special"]), N)
    cases = {
        "too many limbs": lambda: ctx.ntt_fwd(x, 1, nq + 1),
        "zero limbs": lambda: ctx.ntt_fwd(x, 1, 0),
        "negative batch": lambda: ctx.ntt_fwd(x, -1, nq),
        "even galois": lambda: ctx.rotate(y, x, key, 1, nq, 4),
        "galois out of range": lambda: ctx.rotate(y, x, key, 1, nq, 2 * N + 1),
        "in place rotate": lambda: ctx.rotate(x, x, key, 1, nq, 5),
        "no hoisted rotations": lambda: ctx.rotate_hoisted(y, x, [], [], 1, nq),
    }
    silent = []
    for name, f in cases.items():
        try:
            f()
            silent.append(name)
        except HxError as e:
            assert str(e)  # a message, not a bare code
    assert not silent, f"accepted silently: {silent}"


def test_ragged_matrices_and_zero_rotation():
    from test_gpu_helix import backend

    from paper_2512_11135_b200.helix import BSGS, DIAG, ROW

    p, be = backend("c2s")
    rng = np.random.default_rng(77)
    n = be.slots
    lvl = be.max_level
    for rows, cols in ((300, 256), (5, 256), (256, 100), (1, 1)):
        A = rng.normal(0, 0.1, (rows, cols))
        x = rng.uniform(-1, 1, cols)
        d = 1 << max(0, (cols - 1).bit_length())
        for meth in (BSGS, DIAG, ROW):
            M = be.prepare(meth, A, lvl)
            be.gen_rotation_keys(M.rotations())
            v = np.zeros(d)
            v[:cols] = x
            ct = be.encrypt(np.tile(v, n // d), lvl)
            outs, rep = be.matvec(M, ct)
            if meth == ROW:
                y = be.decrypt(outs[0])[:rows]
            else:
                y = np.concatenate([be.decrypt(o)[:d] for o in outs])[:rows]
            assert np.abs(y - A @ x).max() < 1e-5, (rows, cols, meth)
    v = rng.uniform(-1, 1, n)
    ct = be.encrypt(v)
    for k in (0, n, -n, 2 * n):  # identity rotations: no key needed
        assert np.abs(be.decrypt(be.rotate(ct, k)) - v).max() < 1e-5


def test_largest_bsgs_shape_at_n4096():
    """d = 2048 = the slot count at N = 2^12 (n1 = 64, n2 = 32): the widest
    diagonal count the MAC kernel accepts (n1 <= 64), 90 %-pruned to keep
    the host encode short."""
    from test_gpu_helix import backend

    from paper_2512_11135_b200.helix import BSGS

    p, be = backend("c2s")
    n = be.slots
    rng = np.random.default_rng(5)
    d = n
    A = np.zeros((d, d))
    live = rng.choice(d, d // 10, replace=False)
    r = np.arange(d)
    for i in live:
        A[r, (r + i) % d] = rng.normal(0, 0.05, d)
    x = rng.uniform(-1, 1, d)
    lvl = 4
    M = be.prepare(BSGS, A, lvl)
    info = M.info()
    assert info["n1"] * info["n2"] == d and info["nonzero"] == len(live)
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(x, lvl)
    outs, rep = be.matvec(M, ct)
    assert np.abs(be.decrypt(outs[0]) - A @ x).max() < 1e-4


def test_bsgs_more_than_64_baby_steps():
    """d = 8192 at N = 2^14 (BsgsPlan n1 = 128, n2 = 64): the MAC runs in
    chunks of 64 baby steps (mac_chunked); dense and 90 %-pruned."""
    from configs import config1

    from paper_2512_11135_b200.helix import BSGS, Backend, params_json

    p = config1(14)
    be = Backend(params_json(p["logn"], p["chain"], p["special"], p["alpha"], 40), seed=3)
    d = be.slots
    rng = np.random.default_rng(8192)
    A = rng.normal(0, 0.01, (d, d))
    x = rng.uniform(-1, 1, d)
    for prune in (False, True):
        B = A.copy()
        if prune:
            r = np.arange(d)
            for i in rng.choice(d, d - d // 10, replace=False):
                B[r, (r + i) % d] = 0.0
        M = be.prepare(BSGS, B, be.max_level)
        info = M.info()
        assert info["n1"] == 128 and info["n2"] == 64
        be.gen_rotation_keys(M.rotations())
        ct = be.encrypt(x)
        outs, rep = be.matvec(M, ct)
        assert np.abs(be.decrypt(outs[0]) - B @ x).max() < 1e-4
        assert rep["rotations"] == 127 + 63 or prune
    be.close()


@pytest.mark.parametrize("cfg", ["toy", "c2", "c2n16"])
def test_batched_rotation_paths_agree_and_repeat(cfg):
    """hx_rotate (one key over a batch), hx_rotate_multi (a key per
    ciphertext) and hx_rotate_grouped (a key per group) are the same key
    switch launched with different grid shapes (E = batch / E = 1 per key):
    their words must agree, and repeated calls must return identical words --
    a cross-CTA race in an in-place pass shows up here as a few differing
    tiles of the last ciphertexts (a packed-digit experiment failed exactly
    so, only at batch >= 15).  The three take the fused ROW-pass + key
    inner-product kernel; hx_rotate_hoisted (one digit set for all keys) the
    separate ROW pass and inner-product kernels, and must give the same
    words: "c2n16" checks the N = 2^16 tile shape of both."""
    import torch

    from paper_2512_11135_b200 import Context

    if cfg == "toy":  # alpha = 1, dnum = n_q (FP64-class specials)
        from oracle_bindings import find_ntt_primes

        logn = 12
        n = 1 << logn
        chain = find_ntt_primes(1 << 34, 1, 2 * n) + find_ntt_primes(1 << 30, 8, 2 * n)
        special = find_ntt_primes(1 << 36, 1, 2 * n)
        alpha = 1
    elif cfg == "c2n16":
        p = config2(16, 24)
        logn, chain, special, alpha = p["logn"], p["chain"], p["special"], p["alpha"]
    else:
        p = config2(12, 12)
        logn, chain, special, alpha = p["logn"], p["chain"], p["special"], p["alpha"]
    n = 1 << logn
    ctx = Context(logn, chain, special, alpha)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    nq = len(chain) - 1
    ext = nq + len(special)
    g = pow(5, 3, 2 * n)
    # a structurally valid rotation-layout key (values uniform): the paths
    # must agree word for word whatever the key is
    full = len(chain) + len(special)
    dmax = ctx.key_words() // (2 * full * n)  # key layout [dnum_max][2][full][N]
    key = torch.zeros((dmax, 2, full, n), dtype=torch.int64, device="cuda")
    for k, q in enumerate(list(chain) + list(special)):
        key[:, :, k, :] = torch.randint(0, q, (dmax, 2, n), generator=gen, device="cuda")
    del ext
    for B in ((1, 3) if cfg == "c2n16" else (1, 3, 15, 16)):
        cts = torch.empty((B, 2, nq, n), dtype=torch.int64, device="cuda")
        for k, q in enumerate(chain[:nq]):
            cts[:, :, k, :] = torch.randint(0, q, (B, 2, n), generator=gen, device="cuda")
        outs = []
        for rep in range(2):
            o1, o2, o3, o4 = (torch.empty_like(cts) for _ in range(4))
            ctx.rotate(o1, cts, key, B, nq, g)
            ctx.rotate_multi(o2, cts, [key] * B, [g] * B, nq)
            ctx.rotate_grouped(o3, cts, [key], [g], B, nq)
            ctx.rotate_hoisted(o4, cts, [key], [g], B, nq)  # unfused: ROW pass + inner product
            torch.cuda.synchronize()
            assert torch.equal(o1, o2) and torch.equal(o1, o3), (cfg, B, rep)
            assert torch.equal(o1, o4), (cfg, B, rep, "fused vs unfused ROW / inner product")
            outs.append(o1.clone())
        assert torch.equal(outs[0], outs[1]), (cfg, B)
