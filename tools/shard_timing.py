"""single-GPU dry run of bench.sharded_bsgs_bench (world 1, reduced rows so the
unsharded matrix fits one GPU; exercises the shard + reduce + rescale path)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

chain, special = bench.primes()
print(json.dumps(bench.sharded_bsgs_bench(torch, None, chain, special, 0, 1, rows=4096, cols=4096)))
