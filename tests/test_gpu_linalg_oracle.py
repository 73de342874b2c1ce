"""Linear-algebra entry points vs the CPU oracle, WORD FOR WORD (VERDICT r1
"next round" 2): BSGS (multi-block, pruned, stacked, token batch, giant-step
shards), packed-row and ct-ct matmul through helix::GpuLatticeBackend, each
recomputed by the oracle drivers (hxo_matvec_bsgs / hxo_matvec_row /
hxo_matmul_ctct) from the same ciphertext and key words.

Plaintexts on the oracle side are built independently of the product's
device encoder (oracle_pipeline: SPEC packing restated + the host encoder
pinned to the reference + oracle RNS lift / NTT), except where noted for the
largest shapes (there the product's own diagonal words are read back; the
device encoder is pinned to the host encoder in test_gpu_encoder.py).

Shapes: config 1 (N = 2^13); the config-2 prime shape at N = 2^12; and at
N = 2^16: a d = 256 BSGS block at 24 limbs, the config-4 d = 128 matmul at a
4-limb level, and a config-5 slice (4096 columns, 2 row blocks of the
11008 x 4096 weight's shape, 3 limbs) split over 2 giant-step shards.
"""
import numpy as np
import pytest

from configs import config1, config2
from oracle_pipeline import (OracleView, d2h, make_mask, pack_bsgs, pack_bsgs_stacked, pack_rows,
                             scale_double)

pytestmark = pytest.mark.gpu

LAZY = True  # the product's BSGS giant steps: one (lazy) ModDown per output

_cache = {}


def view(name):
    from paper_2512_11135_b200.helix import Backend, params_json

    if name not in _cache:
        p = {"c1": lambda: config1(13), "c2s": lambda: config2(12, 24), "c2": lambda: config2(16, 24),
             "c2q4": lambda: dict(config2(16, 24), chain=config2(16, 24)["chain"][:4]),
             "c2q3": lambda: dict(config2(16, 24), chain=config2(16, 24)["chain"][:3])}[name]()
        be = Backend(params_json(p["logn"], p["chain"], p["special"], p["alpha"], 40), seed=11)
        _cache[name] = OracleView(be, p)
    return _cache[name]


def encode_diags(ov, payloads, level):
    q = float(ov.q(level))
    return [None if v is None else ov.encode(v, level, q) for v in payloads]


def out_words(ov, cts, n_q):
    return np.stack([ov.ct(c, n_q) for c in cts])


# ------------------------------------------------------------------ config 1
@pytest.mark.parametrize("shape", [(64, 64), (128, 64), (40, 64)])
def test_config1_bsgs_words_vs_oracle(shape):
    from paper_2512_11135_b200.helix import BSGS

    ov = view("c1")
    be, N = ov.be, ov.N
    rng = np.random.default_rng(20251211 * 10 + 1)
    A = rng.uniform(-1, 1, shape)
    x = rng.uniform(-1, 1, shape[1])
    lvl = be.max_level
    M = be.prepare(BSGS, A, lvl)
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(np.tile(x, be.slots // 64), lvl)
    outs, rep = be.matvec(M, ct)
    pl, d, n1, n2, blocks = pack_bsgs(A, be.slots)
    assert (d, n1, n2, blocks) == (M.info()["d"], M.info()["n1"], M.info()["n2"], M.info()["blocks"])
    diags = encode_diags(ov, pl, lvl)
    exp = ov.orc.matvec_bsgs(ov.ct(ct), lvl + 1, n1, n2, blocks, diags, ov.keys(M.rotations()), lazy=LAZY)
    assert np.array_equal(out_words(ov, outs, lvl), exp)


def test_config1_row_words_vs_oracle():
    """configs[0] through the packed-row method (the comparison method of the config)"""
    from paper_2512_11135_b200.helix import ROW

    ov = view("c1")
    be = ov.be
    rng = np.random.default_rng(20251211 * 10 + 1)
    A = rng.uniform(-1, 1, (64, 64))
    x = rng.uniform(-1, 1, 64)
    lvl = be.max_level
    M = be.prepare(ROW, A, lvl)
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(np.tile(x, be.slots // 64), lvl)
    outs, rep = be.matvec(M, ct)
    rows_pl, pc, p = pack_rows(A, be.slots)
    rows_pts = [ov.encode(v, lvl, float(ov.q(lvl))) for v in rows_pl]
    masks = []
    for r in range(p):
        m = np.zeros(be.slots)
        m[r * pc] = 1.0
        masks.append(ov.encode(m, lvl - 1, float(ov.q(lvl - 1))))
    exp = ov.orc.matvec_row(ov.ct(ct), lvl + 1, p, A.shape[0], pc, rows_pts, masks, ov.keys(M.rotations()))
    assert np.array_equal(ov.ct(outs[0], lvl - 1), exp)


def _matmul_vs_oracle(ov, d, level, seed):
    be = ov.be
    rng = np.random.default_rng(seed)
    A = rng.normal(0, 1, (d, d))
    B = rng.normal(0, 1, (d, d))
    be.gen_rotation_keys(be.matmul_rotations(d))
    ca = be.encrypt(A.reshape(-1), level)
    cb = be.encrypt(B.reshape(-1), level)
    c, rep = be.matmul(ca, cb, d)
    n = be.slots
    qa, qb = ov.q(level), ov.q(level - 1)
    cm = [ov.encode(make_mask("col", j, d, n), level, float(qa)) for j in range(d)]
    rm = [ov.encode(make_mask("row", j, d, n), level, scale_double(-40, [qa, qb])) for j in range(d)]
    keys = ov.keys(be.matmul_rotations(d))
    exp = ov.orc.matmul_ctct(ov.ct(ca), ov.ct(cb), level + 1, d, cm, rm, ov.rlk(), keys)
    assert np.array_equal(ov.ct(c, level - 1), exp)
    out = be.decrypt(c)[: d * d].reshape(d, d)
    assert np.abs(out - A @ B).max() < 1e-3 * d


@pytest.mark.parametrize("d", [2, 4, 8])
def test_config1_matmul_words_vs_oracle(d):
    ov = view("c1")
    _matmul_vs_oracle(ov, d, ov.be.max_level, d)


# ------------------------------------------------------------------ config-2 primes at N = 2^12
def _launches(be, kernel, fn):
    """fn() with the launches of kernel family `kernel` counted on the backend's context"""
    import ctypes as C

    from paper_2512_11135_b200.hx import lib

    L = lib()
    L.hx_ctx_time_kernel.argtypes = [C.c_void_p, C.c_char_p]
    L.hx_ctx_kernel_time.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
    h = be.device_context()
    assert L.hx_ctx_time_kernel(h, kernel.encode()) == 0
    out = fn()
    ms, n = C.c_double(), C.c_longlong()
    assert L.hx_ctx_kernel_time(h, C.byref(ms), C.byref(n)) == 0
    assert L.hx_ctx_time_kernel(h, None) == 0
    return out, n.value


def _bsgs_case(ov, A, lvl, method_stacked=False, expect_kernel=None):
    from paper_2512_11135_b200.helix import BSGS, BSGS_STACKED

    be = ov.be
    M = be.prepare(BSGS_STACKED if method_stacked else BSGS, A, lvl)
    be.gen_rotation_keys(M.rotations())
    d = M.info()["d"]
    x = np.random.default_rng(7).uniform(-1, 1, A.shape[1])
    v = np.zeros(d)
    v[: A.shape[1]] = x
    ct = be.encrypt(np.tile(v, be.slots // d), lvl)
    if expect_kernel:
        (outs, rep), n = _launches(be, expect_kernel, lambda: be.matvec(M, ct))
        assert n > 0, f"{expect_kernel} did not run"
    else:
        outs, rep = be.matvec(M, ct)
    if method_stacked:
        pl, d2, n1, n2 = pack_bsgs_stacked(A, be.slots)
        blocks = 1
    else:
        pl, d2, n1, n2, blocks = pack_bsgs(A, be.slots)
    assert d2 == d
    diags = encode_diags(ov, pl, lvl)
    exp = ov.orc.matvec_bsgs(ov.ct(ct), lvl + 1, n1, n2, blocks, diags, ov.keys(M.rotations()), lazy=LAZY)
    assert np.array_equal(out_words(ov, outs, lvl), exp)
    return M, ct, diags, exp


@pytest.mark.parametrize("stacked", [False, True])
@pytest.mark.parametrize("prune", [0, 5, 230])
def test_c2s_bsgs_multiblock_words_vs_oracle(stacked, prune):
    """dense (one streaming MAC), mostly dense (5 zero diagonals per block:
    dense giant groups on the streaming MAC, the rest on the index-list MAC)
    and 90 %-pruned (index-list MAC) blocks"""
    ov = view("c2s")
    rng = np.random.default_rng(100 + 2 * stacked + prune)
    A = rng.normal(0, 0.02, (512, 256))
    if prune:  # `prune` generalized diagonals of every block zeroed
        for b in range(2):
            for i in rng.choice(256, prune, replace=False):
                for j in range(256):
                    A[b * 256 + j, (i + j) % 256] = 0
    _bsgs_case(ov, A, ov.be.max_level, stacked)


@pytest.mark.parametrize("n1,expect", [(-1, (32, 8)), (64, (64, 4)), (8, (8, 32))])
def test_c2s_bsgs_explicit_plan_words_vs_oracle(n1, expect):
    """a non-default BSGS split (hxc_matrix_prepare_plan): the cost-tuned one
    (BsgsPlan::for_cost, 3 row blocks of d = 256 -> 32 x 8) and two explicit
    ones, against the oracle driver run with the same n1, n2"""
    from paper_2512_11135_b200.helix import BSGS

    ov = view("c2s")
    be = ov.be
    lvl = be.max_level
    rng = np.random.default_rng(300 + n1)
    A = rng.normal(0, 0.02, (768, 256))
    M = be.prepare(BSGS, A, lvl, n1)
    info = M.info()
    assert (info["n1"], info["n2"], info["blocks"]) == (expect[0], expect[1], 3)
    be.gen_rotation_keys(M.rotations())
    ct = be.encrypt(np.tile(rng.uniform(-1, 1, 256), be.slots // 256), lvl)
    (outs, rep), n_p40 = _launches(be, "bsgs_mac_p40_kernel", lambda: be.matvec(M, ct))
    # n1 in {32, 64}: the three dense blocks go through ONE packed MAC launch
    # (hx_bsgs_mac_p40_blocks: 3 x n2 rows); n1 = 8 takes the streaming u64 MAC
    assert n_p40 == (1 if expect[0] >= 32 else 0)
    assert rep["rotations"] == (expect[0] - 1) + 3 * (expect[1] - 1)
    pl, d, p1, p2, blocks = pack_bsgs(A, be.slots, expect[0])
    diags = encode_diags(ov, pl, lvl)
    exp = ov.orc.matvec_bsgs(ov.ct(ct), lvl + 1, p1, p2, blocks, diags, ov.keys(M.rotations()), lazy=LAZY)
    assert np.array_equal(out_words(ov, outs, lvl), exp)


@pytest.mark.parametrize("prune", [0, 5])
def test_c2s_bsgs_packed_p40_words_vs_oracle(prune):
    """d = 1024 (n1 = n2 = 32), one block of 32 rows, one token: the packed
    5-byte MAC (hx_bsgs_mac_p40) on the dense block, or on the dense giant-group
    runs of a mostly dense block (5 zero diagonals; the rest on the index-list
    MAC) vs the oracle"""
    ov = view("c2s")
    rng = np.random.default_rng(400 + prune)
    A = rng.normal(0, 0.02, (1024, 1024))
    if prune:
        for i in rng.choice(1024, prune, replace=False):
            for j in range(1024):
                A[j, (i + j) % 1024] = 0
    M, *_ = _bsgs_case(ov, A, ov.be.max_level, expect_kernel="bsgs_mac_p40_kernel")
    assert M.info()["n1"] == 32 and M.info()["blocks"] == 1


def test_config1_bsgs_packed_p40_n64_words_vs_oracle():
    """d = 4096 (n1 = n2 = 64) at config 1 (N = 2^13, 3 limbs of 40 bits): the
    packed MAC with 8 baby steps per warp vs the oracle"""
    ov = view("c1")
    rng = np.random.default_rng(401)
    A = rng.normal(0, 0.02, (4096, 4096))
    M, *_ = _bsgs_case(ov, A, ov.be.max_level, expect_kernel="bsgs_mac_p40_kernel")
    assert M.info()["n1"] == 64


@pytest.mark.parametrize("prune", [0, 5])
def test_c2s_bsgs_tensor_core_rows96_words_vs_oracle(prune):
    """6 row blocks x n2 = 16 = 96 rows, n1 = 16, one token: the tensor-core MAC
    path of bsgs_blocks_tokens (all blocks in one hx_bsgs_mac_tc launch;
    absent diagonals as zero operand rows) vs the oracle"""
    ov = view("c2s")
    rng = np.random.default_rng(300 + prune)
    A = rng.normal(0, 0.02, (1536, 256))
    if prune:
        for b in range(6):
            for i in rng.choice(256, prune, replace=False):
                for j in range(256):
                    A[b * 256 + j, (i + j) % 256] = 0
    M, *_ = _bsgs_case(ov, A, ov.be.max_level, expect_kernel="bsgs_mac_tc_kernel")
    assert M.info()["blocks"] == 6 and M.info()["n1"] == 16


def test_c2s_bsgs_token_batch_words_vs_oracle():
    from paper_2512_11135_b200.helix import BSGS

    ov = view("c2s")
    be = ov.be
    rng = np.random.default_rng(8)
    A = rng.normal(0, 0.05, (512, 256))
    lvl = 9
    M = be.prepare(BSGS, A, lvl)
    be.gen_rotation_keys(M.rotations())
    cts = [be.encrypt(np.tile(rng.uniform(-1, 1, 256), be.slots // 256), lvl) for _ in range(4)]
    outs, rep = be.matvec_tokens(M, cts)
    pl, d, n1, n2, blocks = pack_bsgs(A, be.slots)
    diags = encode_diags(ov, pl, lvl)
    keys = ov.keys(M.rotations())
    for t, ct in enumerate(cts):
        exp = ov.orc.matvec_bsgs(ov.ct(ct), lvl + 1, n1, n2, blocks, diags, keys, lazy=LAZY)
        assert np.array_equal(out_words(ov, outs[t], lvl), exp), t


@pytest.mark.parametrize("world", [2, 3])
def test_c2s_giant_step_shards_words_vs_oracle(world):
    """each rank's pre-rescale partials == the oracle over that rank's giant
    range, and the int64 sum + hx_reduce_mod_q + rescale == the oracle's full matvec"""
    import torch

    from paper_2512_11135_b200.helix import BSGS
    from paper_2512_11135_b200.shard import finish, gather_words, reduce_partials, shard_range

    ov = view("c2s")
    be, N = ov.be, ov.N
    rng = np.random.default_rng(30 + world)
    A = rng.normal(0, 0.02, (512, 256))
    lvl = 6
    nq = lvl + 1
    x = rng.uniform(-1, 1, 256)
    ct = be.encrypt(np.tile(x, be.slots // 256), lvl)
    pl, d, n1, n2, blocks = pack_bsgs(A, be.slots)
    diags = encode_diags(ov, pl, lvl)
    M = be.prepare(BSGS, A, lvl)
    be.gen_rotation_keys(M.rotations())
    keys = ov.keys(M.rotations())
    xw = ov.ct(ct)
    total, like = None, None
    for r in range(world):
        Ms = be.prepare_shard(A, lvl, r, world)
        parts, rep = be.matvec_shard(Ms, ct)
        gb, ge = shard_range(n2, r, world)
        exp = ov.orc.matvec_bsgs(xw, nq, n1, n2, blocks, diags, keys, giant=(gb, ge), partial=True)
        pw = be.shard_partial_words(parts[0])
        got = np.stack([d2h(p_.device_ptr(), pw) for p_ in parts])
        assert np.array_equal(got, exp), f"rank {r} partials"
        w = gather_words(parts, pw, torch)
        total = w if total is None else total + w
        like = parts
    torch.cuda.synchronize()
    reduce_partials(be.device_context(), total, blocks, nq, lambda t: None, ov.K, world, ov.chain + ov.special)
    outs = finish(be, like, total)
    exp = ov.orc.matvec_bsgs(xw, nq, n1, n2, blocks, diags, keys, lazy=LAZY)
    assert np.array_equal(out_words(ov, outs, lvl), exp)


# ------------------------------------------------------------------ N = 2^16
@pytest.mark.slow
def test_n16_bsgs_block_24_limbs_words_vs_oracle():
    """a d = 256 BSGS block (n1 = n2 = 16) at the full 24-limb level, N = 2^16"""
    ov = view("c2")
    rng = np.random.default_rng(20251211 * 10 + 3)
    A = rng.normal(0, 0.02, (256, 256))
    _bsgs_case(ov, A, ov.be.max_level)


@pytest.mark.slow
def test_n16_matmul_d128_4_limbs_words_vs_oracle():
    """config 4: Q K^T shape (d = 128 padded) at a 4-limb level, N = 2^16"""
    ov = view("c2q4")
    _matmul_vs_oracle(ov, 128, 3, 20251211 * 10 + 4)


@pytest.mark.slow
def test_n16_config5_slice_shards_words_vs_oracle():
    """config 5's shape on a slice: 8192 x 4096 (d = 4096, n1 = n2 = 64, 2 row
    blocks) at 3 limbs, N = 2^16, split over 2 giant-step shards; partials and
    the reduced, rescaled result vs the oracle (diagonal words read back from
    the product: 8192 host encodes would dominate the test)."""
    import torch

    from paper_2512_11135_b200.helix import BSGS
    from paper_2512_11135_b200.shard import finish, gather_words, reduce_partials, shard_range

    ov = view("c2q3")
    be, N = ov.be, ov.N
    rng = np.random.default_rng(20251211 * 10 + 5)
    A = rng.normal(0, 0.02, (8192, 4096))
    x = rng.uniform(-1, 1, 4096)
    lvl = 2
    nq = 3
    ct = be.encrypt(np.tile(x, be.slots // 4096), lvl)
    xw = ov.ct(ct)
    world = 2
    total, like, keys, diags = None, None, None, {}
    for r in range(world):
        Ms = be.prepare_shard(A, lvl, r, world)
        if keys is None:
            be.gen_rotation_keys(Ms.rotations())
            keys = ov.keys(Ms.rotations())
        info = Ms.info()
        n1, n2, blocks = info["n1"], info["n2"], info["blocks"]
        for i in range(Ms.payload_count()):
            ptr_ = Ms.payload_ptr(i)
            if ptr_:
                diags[i] = d2h(ptr_, nq * N).reshape(nq, N)
        parts, rep = be.matvec_shard(Ms, ct)
        gb, ge = shard_range(n2, r, world)
        dl = [diags.get(i) for i in range(blocks * n1 * n2)]
        exp = ov.orc.matvec_bsgs(xw, nq, n1, n2, blocks, dl, keys, giant=(gb, ge), partial=True)
        pw = be.shard_partial_words(parts[0])
        got = np.stack([d2h(p_.device_ptr(), pw) for p_ in parts])
        assert np.array_equal(got, exp), f"rank {r}"
        w = gather_words(parts, pw, torch)
        total = w if total is None else total + w
        like = parts
        del Ms
    torch.cuda.synchronize()
    reduce_partials(be.device_context(), total, blocks, nq, lambda t: None, ov.K, world, ov.chain + ov.special)
    outs = finish(be, like, total)
    dl = [diags.get(i) for i in range(blocks * n1 * n2)]
    exp = ov.orc.matvec_bsgs(xw, nq, n1, n2, blocks, dl, keys, lazy=LAZY)
    assert np.array_equal(out_words(ov, outs, lvl), exp)
    y = np.concatenate([be.decrypt(o)[:4096] for o in outs])
    assert np.abs(y - A @ x).max() < 1e-4


@pytest.mark.parametrize("name,d,H", [("c1", 8, 3), ("c2s", 16, 4)])
def test_matmul_heads_words_vs_oracle(name, d, H):
    """config 4's head batch (hxc_matmul_heads): every head's output equals the
    single-head product and the oracle's matmul word for word; per-head counters"""
    ov = view(name)
    be = ov.be
    lvl = be.max_level
    rng = np.random.default_rng(90 + d)
    be.gen_rotation_keys(be.matmul_rotations(d))
    As = [rng.normal(0, 1, (d, d)) for _ in range(H)]
    Bs = [rng.normal(0, 1, (d, d)) for _ in range(H)]
    ca = [be.encrypt(A.reshape(-1), lvl) for A in As]
    cb = [be.encrypt(B.reshape(-1), lvl) for B in Bs]
    outs, rep = be.matmul_heads(ca, cb, d)
    lg = d.bit_length() - 1
    assert rep["rotations"] == 2 * d * (1 + lg) - 2 and rep["ct_muls"] == d and rep["levels_consumed"] == 2
    n = be.slots
    qa, qb = ov.q(lvl), ov.q(lvl - 1)
    cm = [ov.encode(make_mask("col", j, d, n), lvl, float(qa)) for j in range(d)]
    rm = [ov.encode(make_mask("row", j, d, n), lvl, scale_double(-40, [qa, qb])) for j in range(d)]
    keys = ov.keys(be.matmul_rotations(d))
    rlk = ov.rlk()
    for h in range(H):
        single, _ = be.matmul(ca[h], cb[h], d)
        got = ov.ct(outs[h], lvl - 1)  # output level lvl - 2: lvl - 1 limbs
        assert np.array_equal(got, ov.ct(single, lvl - 1)), h
        if h in (0, H - 1):
            exp = ov.orc.matmul_ctct(ov.ct(ca[h]), ov.ct(cb[h]), lvl + 1, d, cm, rm, rlk, keys)
            assert np.array_equal(got, exp), h
        dec = be.decrypt(outs[h])[: d * d].reshape(d, d)
        assert np.abs(dec - As[h] @ Bs[h]).max() < 1e-3 * d
