import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2512_11135_b200.helix import Backend, params_json, BSGS
from paper_2512_11135_b200.shard import sharded_matvec, gather_words
chain, special = bench.primes()
be = Backend(params_json(bench.LOGN, chain, special, bench.ALPHA, 40), seed=5)
rng = np.random.default_rng(1)
W = rng.normal(0, 0.02, (4096, 4096)); x = rng.uniform(-1, 1, 4096)
lvl = be.max_level
M = be.prepare_shard(W, lvl, 0, 1); be.gen_rotation_keys(M.rotations())
M2 = be.prepare(BSGS, W, lvl)
ct = be.encrypt(np.tile(x, be.slots // 4096), lvl)
def t(f, n=3):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("matvec full", t(lambda: be.matvec(M2, ct)))
print("matvec_shard", t(lambda: be.matvec_shard(M, ct)))
print("sharded_matvec", t(lambda: sharded_matvec(be, M, ct, lvl + 1, bench.N, lambda x: None, torch)))
