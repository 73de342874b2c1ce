"""CPU (gloo, world_size 2) test of the multi-GPU giant-step sharding math
(paper_2512_11135_b200/shard.py).

Each rank runs the oracle's BSGS driver (hxo_matvec_bsgs) restricted to its
giant groups (shard_range) in PARTIAL mode: with double-hoisted giant steps a
partial is T = [2][n_q][N] plus S = [2][n_q + K][N] (the key-switch products
before their single ModDown).  The ranks all-reduce those words as int64
(the same call shard.sharded_matvec makes over NCCL), reduce T and S mod q,
finish with T + ModDown(S) and rescale once.  The result must equal the
unsharded oracle pipeline word for word.  Keys / diagonals are uniform random
words: bit-exactness of the combination does not depend on them being well
formed.  (The product's own shard path over gloo is tests/test_gpu_shard_mp.py.)
"""
import os
import socket

import numpy as np
import pytest

from configs import config1, config2
from oracle_bindings import Oracle, uniform_limbs

from paper_2512_11135_b200.shard import check_exact_sum, shard_range

CASES = {"c1": dict(logn=10, nq=3, n1=4, n2=4, blocks=2, seed=11),
         "c2": dict(logn=10, nq=6, n1=4, n2=8, blocks=1, seed=12)}


def _params(name):
    c = CASES[name]
    return config1(c["logn"]) if name == "c1" else config2(c["logn"], 8)


def _inputs(orc, p, c):
    N = 1 << p["logn"]
    nq = c["nq"]
    chain = p["chain"][:nq]
    full = p["chain"] + p["special"]
    K = len(p["special"])
    rng = np.random.default_rng(c["seed"])  # identical on every rank
    xw = uniform_limbs(rng, chain, N, (2,))
    dn = orc.dnum(len(p["chain"]))
    keys = {}
    for r in list(range(1, c["n1"])) + [c["n1"] * j for j in range(1, c["n2"])]:
        keys[r] = np.ascontiguousarray(uniform_limbs(rng, full, N, (dn, 2)).reshape(dn, 2, len(full), N))
    diags = [uniform_limbs(rng, chain, N) for _ in range(c["blocks"] * c["n1"] * c["n2"])]
    diags[3] = None  # a zero diagonal
    return xw, keys, diags, K


def _finish(orc, words, p, nq, K, blocks):
    """T + ModDown(S) per block, then rescale (reduced words in)"""
    N = 1 << p["logn"]
    out = []
    for b in range(blocks):
        w = words[b]
        T = w[: 2 * nq * N].reshape(2, nq, N)
        S = np.ascontiguousarray(w[2 * nq * N:].reshape(2, nq + K, N))
        md = orc.moddown_ntt(S, nq, 2)
        y = np.stack([orc.binop("hxo_add", np.ascontiguousarray(T[i]), md[i], nq) for i in range(2)])
        out.append(np.stack([orc.rescale_ntt(np.ascontiguousarray(y[i]), nq) for i in range(2)]))
    return np.stack(out)


def _reduce(words, p, nq, K):
    N = 1 << p["logn"]
    qT = np.array(p["chain"][:nq], dtype=np.uint64)
    qS = np.array(p["chain"][:nq] + p["special"], dtype=np.uint64)
    out = words.view(np.uint64).copy()
    for b in range(out.shape[0]):
        T = out[b, : 2 * nq * N].reshape(2, nq, N)
        S = out[b, 2 * nq * N:].reshape(2, nq + K, N)
        T %= qT[None, :, None]
        S %= qS[None, :, None]
    return out


def _worker(rank, world, port, out_dir, name):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = CASES[name]
        p = _params(name)
        orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
        nq = c["nq"]
        xw, keys, diags, K = _inputs(orc, p, c)
        gb, ge = shard_range(c["n2"], rank, world)
        part = orc.matvec_bsgs(xw, nq, c["n1"], c["n2"], c["blocks"], diags, keys, giant=(gb, ge), partial=True)
        check_exact_sum(world, p["chain"] + p["special"])
        t = torch.from_numpy(part.view(np.int64).copy())
        dist.all_reduce(t)  # int64 wrap sum == exact u64 sum (world * q < 2^64)
        summed = _reduce(t.numpy(), p, nq, K)
        out = _finish(orc, summed, p, nq, K, c["blocks"])
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), out)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for n2 in (1, 2, 5, 16, 33):
        for world in (1, 2, 3, 4, 8):
            got = [shard_range(n2, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n2
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_exact_sum_guard():
    check_exact_sum(8, [(1 << 60) - 1])
    with pytest.raises(ValueError):
        check_exact_sum(8, [(1 << 62) - 57])  # 8 (q - 1) >= 2^64 would wrap silently


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_giant_step_shards_gloo_world2(tmp_path, name):
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), name), nprocs=world, start_method="spawn")
    c = CASES[name]
    p = _params(name)
    orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
    xw, keys, diags, K = _inputs(orc, p, c)
    ref = orc.matvec_bsgs(xw, c["nq"], c["n1"], c["n2"], c["blocks"], diags, keys, lazy=True)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.array_equal(got, ref), f"rank {r} differs from the unsharded pipeline"
