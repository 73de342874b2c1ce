"""GPU tests of the helix SlotBackend on B200 (libhelix_b200.so via helix_c.h):
CKKS round trips and the SPEC known answers on the lattice backend, the
linear-algebra entry points vs cleartext within the stated CKKS error bound,
trace counts equal to the SPEC closed forms, and the BSGS matvec ciphertext
bit-exact against the CPU oracle recomputing the same pipeline from the same
words (input ciphertext, keys, encoded diagonals).
"""
import ctypes as C

import numpy as np
import pytest

from configs import config1, config2
from oracle_bindings import Oracle, galois_elt

pytestmark = pytest.mark.gpu

# decrypt error bound (absolute, slots in [-1, 1]); measured ~1e-7 at Delta = 2^40
TOL = 1e-4

_cache = {}


def backend(name):
    """c1 / c2s; a "+ck" suffix selects compressed key storage (compress_keys)"""
    from paper_2512_11135_b200.helix import Backend, params_json

    if name not in _cache:
        base = name.split("+")[0]
        p = config1(13) if base == "c1" else config2(12, 24)
        extra = {"compress_keys": True} if name.endswith("+ck") else {}
        be = Backend(params_json(p["logn"], p["chain"], p["special"], p["alpha"], 40, **extra), seed=7)
        _cache[name] = (p, be)
    return _cache[name]


def d2h(ptr, words):
    from paper_2512_11135_b200.hx import lib

    out = np.zeros(words, dtype=np.uint64)
    L = lib()
    L.hx_memcpy_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    L.hx_stream_sync.argtypes = [C.c_void_p]
    assert L.hx_device_sync() == 0
    assert L.hx_memcpy_d2h(out.ctypes.data, ptr, words * 8, None) == 0
    assert L.hx_stream_sync(None) == 0
    return out


@pytest.mark.parametrize("name", ["c1", "c2s"])
def test_roundtrip_rotate_mul(name):
    p, be = backend(name)
    n = be.slots
    rng = np.random.default_rng(1)
    m = rng.uniform(-1, 1, n)
    ct = be.encrypt(m)
    assert np.abs(be.decrypt(ct) - m).max() < TOL
    be.gen_rotation_keys([1, 5, n // 2])
    for k in (1, 5, n // 2):
        assert np.abs(be.decrypt(be.rotate(ct, k)) - np.roll(m, -k)).max() < TOL
    # relinearised square of [2,3] -> [4,9]
    sq = be.rescale(be.mul(be.encrypt([2.0, 3.0]), be.encrypt([2.0, 3.0])))
    out = be.decrypt(sq)
    assert abs(out[0] - 4) < 1e-3 and abs(out[1] - 9) < 1e-3
    assert sq.level == be.max_level - 1
    # rescale preserves values
    pm = be.rescale(be.mul_plain(ct, np.ones(n)))
    assert np.abs(be.decrypt(pm) - m).max() < TOL
    # composition Rot(Rot(x,1),5) = Rot(x,6) within 1e-3
    be.gen_rotation_keys([6])
    assert np.abs(be.decrypt(be.rotate(be.rotate(ct, 1), 5)) - be.decrypt(be.rotate(ct, 6))).max() < 1e-3


def test_errors_map_to_reference_types():
    from paper_2512_11135_b200.hx import HxError

    p, be = backend("c1")
    ct = be.encrypt([1.0])
    with pytest.raises(HxError, match="no key for amount"):
        be.rotate(ct, 7)
    with pytest.raises(HxError, match="level mismatch"):
        be.add(ct, be.mod_down(ct, 0))
    with pytest.raises(HxError, match="scale not above Delta"):
        be.rescale(ct)


@pytest.mark.parametrize("method", ["bsgs", "diag", "row"])
def test_config1_matvec_64x64(method):
    """BASELINE configs[0]: 64x64 U[-1,1] matrix and vector, one ciphertext."""
    from paper_2512_11135_b200.helix import BSGS, DIAG, ROW

    p, be = backend("c1")
    rng = np.random.default_rng(20251211 * 10 + 1)
    A = rng.uniform(-1, 1, (64, 64))
    x = rng.uniform(-1, 1, 64)
    meth = {"bsgs": BSGS, "diag": DIAG, "row": ROW}[method]
    M = be.prepare(meth, A, be.max_level)
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(np.tile(x, be.slots // 64))
    be.trace_reset()
    outs, rep = be.matvec(M, ct)
    y = be.decrypt(outs[0])[:64]
    assert np.abs(y - A @ x).max() < 1e-2 * 0 + 1e-5 * 64
    tr = be.trace()["counts"]
    assert tr["rotate"] == rep["rotations"]
    if method == "bsgs":
        assert rep["rotations"] == 14 and rep["levels_consumed"] == 1 and rep["pt_muls"] == 64
    if method == "diag":
        assert rep["rotations"] == 63 and rep["levels_consumed"] == 1
    if method == "row":
        assert rep["levels_consumed"] == 2 and rep["rotations"] == 6 + 63
    assert abs(rep["output_scale_log2"] - 40.0) < 1e-12


@pytest.mark.parametrize("keys", ["full", "compressed"])
def test_bsgs_matvec_bit_exact_vs_oracle(keys):
    """The fused BSGS pipeline (hoisted baby steps, streaming MAC, batched giant
    rotations with one lazy ModDown, rescale) reproduces the oracle's
    ciphertext word for word, with full and with compressed (seeded) key
    storage."""
    from paper_2512_11135_b200.helix import BSGS

    p, be = backend("c1" if keys == "full" else "c1+ck")
    n, N, nq, K = be.slots, 1 << p["logn"], 3, 1
    orc = Oracle(p["logn"], p["chain"], p["special"], 1)
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (64, 64))
    x = rng.uniform(-1, 1, 64)
    M = be.prepare(BSGS, A, 2)
    info = M.info()
    n1, n2 = info["n1"], info["n2"]
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(np.tile(x, n // 64))
    outs, rep = be.matvec(M, ct)
    got = d2h(outs[0].device_ptr(), 2 * (nq - 1) * N).reshape(2, nq - 1, N)
    # the same words, recomputed on the CPU oracle
    xw = d2h(ct.device_ptr(), 2 * nq * N).reshape(2, nq, N)
    kw = orc.dnum(nq) * 2 * (nq + K) * N

    def std_key(k):
        import torch

        g = galois_elt(k, N)
        full = torch.empty(kw, dtype=torch.int64, device="cuda")
        be.expand_key(be.rotation_key_ptr(k), full.data_ptr())  # the backend stores compressed keys
        rot = d2h(full.data_ptr(), kw).reshape(-1, N)
        # rotation layout = tau_{g^-1}(standard)  =>  standard = tau_g(rotation layout)
        return np.ascontiguousarray(orc.automorphism_ntt(rot, rot.shape[0], 0, g).reshape(orc.dnum(nq), 2, nq + K, N))

    diags = [d2h(M.payload_ptr(i), nq * N).reshape(nq, N) for i in range(64)]
    keys = {k: std_key(k) for k in list(range(1, n1)) + [n1 * j for j in range(1, n2)]}
    # baby steps hoisted, MAC, giant steps double hoisted (one ModDown), rescale
    exp = orc.matvec_bsgs(xw, nq, n1, n2, 1, diags, keys, lazy=True)[0]
    assert np.array_equal(got, exp)


def test_multiblock_bsgs_and_sparse_config2_shape():
    """config-2 prime shape (24+3 primes, alpha=3) at N=2^12: a 512x256 matrix
    (2 row blocks, baby steps shared) and a 90%-pruned variant."""
    from paper_2512_11135_b200.helix import BSGS

    p, be = backend("c2s")
    rng = np.random.default_rng(3)
    A = rng.normal(0, 0.02, (512, 256))
    x = rng.uniform(-1, 1, 256)
    lvl = be.max_level
    for prune in (False, True):
        B = A.copy()
        if prune:  # zero 90% of the generalized diagonals (per block)
            for b in range(2):
                for i in rng.choice(256, 230, replace=False):
                    for j in range(256):
                        B[b * 256 + j, (i + j) % 256] = 0
        M = be.prepare(BSGS, B, lvl)
        be.gen_rotation_keys(M.rotations())
        ct = be.encrypt(np.tile(x, be.slots // 256), lvl)
        outs, rep = be.matvec(M, ct)
        y = np.concatenate([be.decrypt(o)[:256] for o in outs])
        assert len(outs) == 2
        assert np.abs(y - B @ x).max() < 1e-5
        if not prune:
            assert rep["rotations"] == 15 + 2 * 15 and rep["pt_muls"] == 512
        else:
            assert rep["pt_muls"] == M.info()["nonzero"] == 2 * 26


@pytest.mark.parametrize("d", [2, 4, 8])
def test_matmul_ctct(d):
    p, be = backend("c1")
    rng = np.random.default_rng(d)
    A = rng.normal(0, 1, (d, d))
    Bm = rng.normal(0, 1, (d, d))
    be.gen_rotation_keys(be.matmul_rotations(d))
    ca = be.encrypt(A.reshape(-1))
    cb = be.encrypt(Bm.reshape(-1))
    c, rep = be.matmul(ca, cb, d)
    lg = d.bit_length() - 1
    assert rep["rotations"] == 2 * d * (1 + lg) - 2 and rep["ct_muls"] == d and rep["pt_muls"] == 2 * d
    assert rep["levels_consumed"] == 2 and abs(rep["output_scale_log2"] - 40) < 1e-12
    out = be.decrypt(c)[: d * d].reshape(d, d)
    assert np.abs(out - A @ Bm).max() < 1e-3 * d


@pytest.mark.parametrize("world,stacked", [(2, False), (3, False), (4, False), (2, True), (3, True)])
def test_giant_step_shards_bit_exact(world, stacked):
    """the G rank shards of a multi-block BSGS matvec (each rank
    its giant groups, pre-rescale partials), summed as int64 words (what the
    NCCL all-reduce does), reduced mod q on the device (hx_reduce_mod_q) and
    rescaled once, equal the single-GPU matvec word for word.  The ranks run
    one after another on this GPU; nothing waits on another rank.  Stacked:
    the same over the stacked-block layout (one output ciphertext)."""
    import torch

    from paper_2512_11135_b200.helix import BSGS, BSGS_STACKED
    from paper_2512_11135_b200.shard import finish, gather_words, reduce_partials, shard_range

    p, be = backend("c2s")
    N = 1 << p["logn"]
    rng = np.random.default_rng(40 + world)
    A = rng.normal(0, 0.02, (512, 256))
    x = rng.uniform(-1, 1, 256)
    lvl = 6
    nq = lvl + 1
    M = be.prepare(BSGS_STACKED if stacked else BSGS, A, lvl)
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(np.tile(x, be.slots // 256), lvl)
    ref, rep_full = be.matvec(M, ct)
    nout = len(ref)
    assert nout == (1 if stacked else 2)
    n2 = M.info()["n2"]
    total = None
    rots = 0
    for r in range(world):
        Ms = be.prepare_shard(A, lvl, r, world, stacked=stacked)
        gb, ge = shard_range(n2, r, world)
        parts, rep = be.matvec_shard(Ms, ct)
        assert len(parts) == nout and rep["levels_consumed"] == 0
        rots += rep["rotations"] - (M.info()["n1"] - 1)  # baby steps are replicated per rank
        w = gather_words(parts, be.shard_partial_words(parts[0]), torch)
        total = w if total is None else total + w  # int64 wrap == u64 sum
        like = parts
    torch.cuda.synchronize()
    reduce_partials(be.device_context(), total, nout, nq, lambda t: None, len(p["special"]), world,
                    p["chain"] + p["special"])
    outs = finish(be, like, total)
    for i in range(nout):
        got = d2h(outs[i].device_ptr(), 2 * lvl * N)
        exp = d2h(ref[i].device_ptr(), 2 * lvl * N)
        assert np.array_equal(got, exp)
    assert rots == rep_full["rotations"] - (M.info()["n1"] - 1)
    if stacked:
        y = be.decrypt(outs[0])[:512]
    else:
        y = np.concatenate([be.decrypt(o)[:256] for o in outs])
    assert np.abs(y - A @ x).max() < 1e-5


@pytest.mark.parametrize("name,shape", [("c1", (64, 64)), ("c2s", (512, 256))])
def test_bsgs_token_batch_matches_single(name, shape):
    """config 3 token batching (helix::matvec_bsgs_tokens): T ciphertexts
    through one matrix with the key switches batched over tokens give the
    same words as T separate matvecs, and per-token counters."""
    from paper_2512_11135_b200.helix import BSGS

    p, be = backend(name)
    N = 1 << p["logn"]
    rows, cols = shape
    rng = np.random.default_rng(rows + 5)
    A = rng.normal(0, 0.05, (rows, cols))
    lvl = be.max_level
    M = be.prepare(BSGS, A, lvl)
    be.gen_rotation_keys(M.rotations())
    xs = [rng.uniform(-1, 1, cols) for _ in range(3)]
    cts = [be.encrypt(np.tile(x, be.slots // cols), lvl) for x in xs]
    outs_t, rep_t = be.matvec_tokens(M, cts)
    nq = lvl  # output level lvl - 1
    for t, ct in enumerate(cts):
        outs_1, rep_1 = be.matvec(M, ct)
        assert rep_t == rep_1
        assert len(outs_t[t]) == len(outs_1)
        for a, b in zip(outs_t[t], outs_1):
            assert np.array_equal(d2h(a.device_ptr(), 2 * nq * N), d2h(b.device_ptr(), 2 * nq * N))
        y = np.concatenate([be.decrypt(o)[:cols] for o in outs_t[t]])[:rows]
        assert np.abs(y - A @ xs[t]).max() < 1e-5


@pytest.mark.parametrize("prune", [False, True])
def test_bsgs_stacked_blocks(prune):
    """Stacked-block BSGS (helix::pack_bsgs_stacked): the 2 row blocks of a
    512 x 256 matrix in one set of full-length diagonals -> one output
    ciphertext with y[row] in slot row, (n1 - 1) + (n2 - 1) rotations and d
    plaintext products; matches the cleartext product and the per-block
    BSGS method."""
    from paper_2512_11135_b200.helix import BSGS, BSGS_STACKED, predicted_rotations

    p, be = backend("c2s")
    rng = np.random.default_rng(512 + prune)
    A = rng.normal(0, 0.02, (512, 256))
    if prune:
        for b in range(2):
            for i in rng.choice(256, 230, replace=False):
                for j in range(256):
                    A[b * 256 + j, (i + j) % 256] = 0
    x = rng.uniform(-1, 1, 256)
    lvl = be.max_level
    M = be.prepare(BSGS_STACKED, A, lvl)
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(np.tile(x, be.slots // 256), lvl)
    be.trace_reset()
    outs, rep = be.matvec(M, ct)
    assert len(outs) == 1
    y = be.decrypt(outs[0])[:512]
    assert np.abs(y - A @ x).max() < 1e-5
    info = M.info()
    if not prune:
        assert rep["rotations"] == 15 + 15 == predicted_rotations(BSGS_STACKED, 512, 256, be.slots)
        assert rep["pt_muls"] == 256
    assert rep["levels_consumed"] == 1 and abs(rep["output_scale_log2"] - 40.0) < 1e-12
    # the per-block method agrees
    M2 = be.prepare(BSGS, A, lvl)
    be.gen_rotation_keys(M2.rotations())
    outs2, rep2 = be.matvec(M2, ct)
    y2 = np.concatenate([be.decrypt(o)[:256] for o in outs2])
    assert np.abs(y - y2).max() < 1e-6
    assert rep["rotations"] <= rep2["rotations"]
