import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import bench
from paper_2512_11135_b200.helix import BSGS, Backend, params_json
chain, special = bench.primes()
be = Backend(params_json(bench.LOGN, chain, special, bench.ALPHA, 40), seed=3)
rng = np.random.default_rng(1)
M = rng.normal(0, 0.02, (3072, 768))
t = time.perf_counter(); mat = be.prepare(BSGS, M, be.max_level); torch.cuda.synchronize(); print("prepare", time.perf_counter() - t)
t = time.perf_counter(); be.gen_rotation_keys(mat.rotations()); torch.cuda.synchronize(); print("keys", time.perf_counter() - t)
