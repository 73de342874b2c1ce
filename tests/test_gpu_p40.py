"""Packed single-token BSGS MAC (hx_bsgs_p40_pack + hx_bsgs_mac_p40: 5-byte
diagonal words streamed by cp.async.bulk, FP64 k-split arithmetic) vs the
CUDA-core MAC over the u64 words (hx_bsgs_mac_tokens) and vs the CPU oracle's
MAC (hxo_bsgs_mac, the mul_acc loop of matvec_bsgs), word for
word: every n1 the kernel takes (32, 64), blocks whose giant groups
are further apart than n1 (diag_jstride), n2 not a multiple of the stage
ring, odd row counts (one row per step) and even ones (two rows per step,
bsgs_mac_p40x_kernel), the 60-bit q_0 on the integer kernel, and the FFN
shapes at N = 2^16."""
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


def run_case(name, n1, n2, dj, seed, oracle_limbs=None):
    import torch

    p, ctx = env(name)
    nq, N = len(p["chain"]), ctx.n
    ctw = 2 * nq * N
    n_diag = (n2 - 1) * dj + n1
    diags = uniform(ctx, nq, n_diag, seed)
    baby = uniform(ctx, nq, n1 * 2, seed + 1).view(n1, 2, nq, N)
    packed = ctx.bsgs_p40_pack(diags, nq, n1, n2, nq, diag_jstride=dj)
    inner = torch.full((n2, 2, nq, N), -1, dtype=torch.int64, device="cuda")
    ctx.bsgs_mac_p40(inner, ctw, baby, packed, diags, nq, n1, n2, nq, diag_jstride=dj)
    ref = torch.empty_like(inner)
    ctx.bsgs_mac_tokens(ref, ctw, 0, baby, 0, diags, nq, n1, n2, nq, tokens=1, diag_jstride=dj)
    got = host(inner)
    assert np.array_equal(got, host(ref)), "P40 MAC != CUDA-core MAC"
    dh, bh = host(diags), host(baby)
    sel = np.concatenate([np.arange(j * dj, j * dj + n1) for j in range(n2)])
    for k in (range(nq) if oracle_limbs is None else oracle_limbs):
        o1 = Oracle(p["logn"], [p["chain"][k]], [], 1)
        exp = o1.bsgs_mac(np.ascontiguousarray(bh[:, :, k:k + 1, :]), np.ascontiguousarray(dh[sel, k:k + 1, :]),
                          n1, n2, 1)
        assert np.array_equal(got[:, :, k:k + 1, :], exp), k


@pytest.mark.parametrize("n1,n2,dj", [(32, 3, 32), (32, 32, 32), (64, 9, 64), (32, 5, 40), (64, 1, 64),
                                       # even row counts: the two-rows-per-step kernel (1 / 2 / 3 / 5 steps; a
                                       # giant-group stride wider than n1)
                                       (32, 2, 32), (64, 4, 64), (64, 6, 80), (32, 10, 32)])
def test_p40_mac_n12_vs_oracle(n1, n2, dj):
    run_case("c2s", n1, n2, dj, 100 + n1 + n2)


def test_p40_mac_config1_shape():
    run_case("c1", 32, 4, 32, 7)


def test_p40_mac_ffn_shapes_n16():
    """the W1 block (n1 = n2 = 32) and the W2 / config-5 block prefix (n1 = 64)
    at N = 2^16, 24 limbs: every word vs the CUDA-core MAC, limbs 0, 1, 23 vs
    the oracle"""
    run_case("c2", 32, 32, 32, 11, oracle_limbs=[0, 1, 23])
    run_case("c2", 64, 12, 64, 12, oracle_limbs=[0, 5])


def test_p40_unsupported_shapes():
    from paper_2512_11135_b200.hx import HxError

    p, ctx = env("c2s")
    import torch

    d = torch.zeros((48, 24, ctx.n), dtype=torch.int64, device="cuda")
    with pytest.raises(HxError):
        ctx.bsgs_p40_pack(d, 24, 16, 3, 24)  # n1 = 16 not in {32, 64}
