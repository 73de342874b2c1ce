"""time the single-GPU stacked config-5 extra alone"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

chain, special = bench.primes()
print(json.dumps(bench.config5_stacked_bench(torch, chain, special)))
