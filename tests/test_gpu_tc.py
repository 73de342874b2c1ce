"""Tensor-core BSGS MAC (hx_bsgs_tc_pack + hx_bsgs_mac_tc, tcgen05.mma kind::i8
on byte-sliced words) vs the CPU oracle's MAC (hxo_bsgs_mac, the mul_acc loop
of matvec_bsgs) and vs the CUDA-core MAC kernels
(hx_bsgs_mac_tokens), word for word.

Shapes: all rows of several row blocks in one launch (rows = blocks * n2 <=
128), T tokens split into launches of 8 / 4 / 2 / 1, absent (zero) diagonals,
the 60-bit q_0 on the integer path beside the 40-bit limbs on the tensor
cores; N = 2^12 / 2^13 (every word vs the oracle) and the FFN W1 shape at
N = 2^16 (sampled limbs vs the oracle, all words vs the CUDA-core MAC)."""
import numpy as np
import pytest

from configs import config1, config2
from oracle_bindings import Oracle

pytestmark = pytest.mark.gpu

_cache = {}


def env(name):
    if name not in _cache:
        from paper_2512_11135_b200 import Context

        p = {"c2": lambda: config2(16, 24), "c2s": lambda: config2(12, 24), "c1": lambda: config1(13)}[name]()
        _cache[name] = (p, Context(p["logn"], p["chain"], p["special"], p["alpha"]))
    return _cache[name]


def host(t):
    import torch

    torch.cuda.synchronize()
    return np.ascontiguousarray(t.cpu().numpy().view(np.uint64))


def uniform(ctx, nq, copies, seed):
    import torch

    t = torch.empty((copies, nq, ctx.n), dtype=torch.int64, device="cuda")
    ctx.sample_uniform(t, nq, 0, copies, seed)
    return t


def run_case(name, blocks, n1, n2, T, zero_frac, seed, oracle_limbs=None):
    import torch

    p, ctx = env(name)
    nq, N = len(p["chain"]), ctx.n
    ctw = 2 * nq * N
    rows = blocks * n2
    rng = np.random.default_rng(seed)
    diags = uniform(ctx, nq, rows * n1, seed).view(blocks, n2 * n1, nq, N)
    live = rng.random(rows * n1) >= zero_frac
    ptrs = [diags[r // n2, (r % n2) * n1 + k].data_ptr() if live[r * n1 + k] else None
            for r in range(rows) for k in range(n1)]
    if live.all():
        dense = diags
    else:
        dense = torch.where(torch.from_numpy(live.reshape(blocks, n2 * n1, 1, 1)).cuda(), diags,
                            torch.zeros_like(diags))
    packed = ctx.bsgs_tc_pack(ptrs, rows, n1, nq)
    baby = uniform(ctx, nq, T * n1 * 2, seed + 1).view(T, n1, 2, nq, N)
    # inner layout of bsgs_blocks_tokens: [n2][T][blocks][2][n_q][N]
    inner = torch.full((n2, T, blocks, 2, nq, N), -1, dtype=torch.int64, device="cuda")
    ctx.bsgs_mac_tc(inner, T * blocks * ctw, ctw, blocks * ctw, baby, n1 * ctw, packed, blocks, n2, n1, nq, tokens=T)
    ref = torch.empty_like(inner)
    for b in range(blocks):
        ctx.bsgs_mac_tokens(ref[:, :, b], T * blocks * ctw, blocks * ctw, baby, n1 * ctw, dense[b], nq, n1, n2, nq,
                            tokens=T)
    got = host(inner)
    assert np.array_equal(got, host(ref)), "tensor-core MAC != CUDA-core MAC"
    limbs = range(nq) if oracle_limbs is None else oracle_limbs
    dh = host(dense)
    bh = host(baby)
    for k in limbs:
        o1 = Oracle(p["logn"], [p["chain"][k]], [], 1)
        for b in range(blocks):
            dk = np.ascontiguousarray(dh[b, :, k:k + 1, :])
            for t in sorted({0, T - 1}):
                bk = np.ascontiguousarray(bh[t, :, :, k:k + 1, :])
                exp = o1.bsgs_mac(bk, dk, n1, n2, 1)
                assert np.array_equal(got[:, t, b, :, k:k + 1, :], exp), (k, b, t)


@pytest.mark.parametrize("blocks,n1,n2,T,zero", [(3, 32, 32, 1, 0.0), (3, 32, 32, 11, 0.1), (2, 64, 64, 2, 0.0),
                                                 (1, 16, 8, 3, 0.3)])
def test_tc_mac_n12_all_limbs(blocks, n1, n2, T, zero):
    """24 + 3 primes at N = 2^12 (q_0 60-bit on the integer path): every limb,
    first and last token, every block vs the oracle"""
    run_case("c2s", blocks, n1, n2, T, zero, 100 + T, oracle_limbs=[0, 1, 7, 23])


def test_tc_mac_config1_shape():
    """config 1 (N = 2^13, 3 x 40-bit chain primes, all on the tensor cores):
    the d = 64 BSGS block n1 = n2 = 8"""
    run_case("c1", 1, 8, 8, 1, 0.0, 7)


def test_tc_mac_w1_n16():
    """FFN W1 at N = 2^16: 3 blocks x n2 = 32 rows, n1 = 32, 24 limbs, 3 tokens"""
    import torch

    torch.cuda.empty_cache()
    run_case("c2", 3, 32, 32, 3, 0.0, 9, oracle_limbs=[0, 13])
    torch.cuda.empty_cache()
