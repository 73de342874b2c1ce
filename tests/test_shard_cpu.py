"""CPU (gloo, world_size 2) test of the multi-GPU giant-step sharding math
(paper_2512_11135_b200/shard.py).

Each rank runs the oracle's BSGS pipeline restricted to its giant groups
(shard_range), produces PRE-RESCALE partials, all-reduces their words as
int64 (the same call bench/sharded_matvec makes over NCCL), reduces mod q and
rescales once.  The result must equal the unsharded oracle pipeline word for
word.  Keys/diagonals are uniform random words: bit-exactness of the
combination does not depend on them being well formed.
"""
import os
import socket

import numpy as np
import pytest

from configs import config1
from oracle_bindings import Oracle, galois_elt, uniform_limbs

from paper_2512_11135_b200.shard import shard_range


def _bsgs_partial(orc, p, nq, n1, n2, gb, ge, seed):
    """oracle BSGS over giant groups [gb, ge) -> (2, nq, N) pre-rescale sum"""
    N = 1 << p["logn"]
    chain = p["chain"][:nq]
    K = len(p["special"])
    full = chain + p["special"]
    rng = np.random.default_rng(seed)  # identical on every rank
    xw = uniform_limbs(rng, chain, N, (2,))
    dn = orc.dnum(nq)

    def key():
        return np.ascontiguousarray(uniform_limbs(rng, full, N, (dn, 2)).reshape(dn, 2, nq + K, N))

    baby_keys = [key() for _ in range(1, n1)]
    giant_keys = [key() for _ in range(1, n2)]
    diags = uniform_limbs(rng, chain, N, (n1 * n2,))
    baby = np.concatenate([xw[None], orc.rotate_hoisted(xw, baby_keys, [galois_elt(k, N) for k in range(1, n1)], nq)])
    inner = orc.bsgs_mac(np.ascontiguousarray(baby), diags, n1, n2, nq)
    acc = np.zeros((2, nq, N), dtype=np.uint64)
    for j in range(gb, ge):
        r = inner[j] if j == 0 else orc.rotate(np.ascontiguousarray(inner[j]), giant_keys[j - 1], nq,
                                               galois_elt(n1 * j, N))
        acc = np.stack([orc.binop("hxo_add", acc[c], r[c], nq) for c in range(2)])
    return acc


def _rescale(orc, acc, nq):
    return np.stack([orc.rescale_ntt(np.ascontiguousarray(acc[c]), nq) for c in range(2)])


def _mod_q(words, chain):
    q = np.array(chain, dtype=np.uint64)[None, :, None]
    return (words.view(np.uint64) % q).astype(np.uint64)


CASE = dict(logn=10, nq=3, n1=4, n2=4, seed=11)


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = config1(CASE["logn"])
        orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
        nq = CASE["nq"]
        gb, ge = shard_range(CASE["n2"], rank, world)
        part = _bsgs_partial(orc, p, nq, CASE["n1"], CASE["n2"], gb, ge, CASE["seed"])
        t = torch.from_numpy(part.view(np.int64).copy())
        dist.all_reduce(t)  # int64 wrap sum == exact u64 sum (world * q < 2^64)
        summed = _mod_q(t.numpy(), p["chain"][:nq])
        out = _rescale(orc, summed, nq)
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


def test_giant_step_shards_gloo_world2(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    p = config1(CASE["logn"])
    orc = Oracle(p["logn"], p["chain"], p["special"], p["alpha"])
    nq = CASE["nq"]
    ref = _rescale(orc, _bsgs_partial(orc, p, nq, CASE["n1"], CASE["n2"], 0, CASE["n2"], CASE["seed"]), nq)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.array_equal(got, ref), f"rank {r} differs from the unsharded pipeline"
