"""The PRODUCT's giant-step sharding path across processes (VERDICT r1
"next round" 10): two processes on this one GPU, each with its own
GpuLatticeBackend (same seed -> same keys and ciphertext words), run
hxc_matrix_prepare_shard / hxc_matvec_shard for their giant groups and
exchange the PQ-basis partials through a gloo all-reduce of host copies
(shard.sharded_matvec with a host-side allreduce); each rank's finished,
rescaled output must equal the unsharded single-process matvec word for word.
The ranks never wait on one another on the device: all synchronisation is in
gloo on the host, after each rank's kernels have completed."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, stacked):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import torch
    import torch.distributed as dist

    from configs import config2
    from paper_2512_11135_b200.helix import BSGS, BSGS_STACKED, Backend, params_json
    from paper_2512_11135_b200.shard import sharded_matvec
    from oracle_pipeline import d2h

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        p = config2(12, 24)
        N = 1 << p["logn"]
        be = Backend(params_json(p["logn"], p["chain"], p["special"], p["alpha"], 40), seed=21)
        rng = np.random.default_rng(5)
        A = rng.normal(0, 0.02, (512, 256))
        x = rng.uniform(-1, 1, 256)
        lvl = 7
        ct = be.encrypt(np.tile(x, be.slots // 256), lvl)  # same RNG sequence on every rank
        M = be.prepare(BSGS_STACKED if stacked else BSGS, A, lvl)
        be.gen_rotation_keys(M.rotations())
        Ms = be.prepare_shard(A, lvl, rank, world, stacked=stacked)

        def host_allreduce(t):  # the exchange over gloo on host copies
            h = t.cpu()
            dist.all_reduce(h)
            t.copy_(h.to(t.device))

        outs, rep = sharded_matvec(be, Ms, ct, lvl + 1, len(p["special"]), host_allreduce, torch, world,
                                   p["chain"] + p["special"])
        ref, _ = be.matvec(M, ct)
        got = np.stack([d2h(o.device_ptr(), 2 * lvl * N) for o in outs])
        exp = np.stack([d2h(o.device_ptr(), 2 * lvl * N) for o in ref])
        xw = d2h(ct.device_ptr(), 2 * (lvl + 1) * N)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), got=got, exp=exp, x=xw,
                 rot=np.array([rep["rotations"]]))
        be.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stacked", [False, True])
def test_product_shards_two_processes_gloo(tmp_path, stacked):
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), stacked), nprocs=world,
                       start_method="spawn")
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    assert np.array_equal(r0["x"], r1["x"]), "ranks must start from the same ciphertext words"
    assert np.array_equal(r0["got"], r0["exp"]), "rank 0: sharded != unsharded"
    assert np.array_equal(r1["got"], r0["exp"]), "rank 1: sharded != unsharded"
