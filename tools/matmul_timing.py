"""time the config-4 matmul extra alone (bench.matmul_bench)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

chain, special = bench.primes()
print(bench.matmul_bench(torch, chain, special))
