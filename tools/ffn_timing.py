"""time the config-3 FFN extras alone (bench.ffn_bsgs_bench)"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--no-w2", action="store_true")
ap.add_argument("--only", nargs="*", default=None)
ap.add_argument("--verbose", action="store_true")
args = ap.parse_args()
chain, special = bench.primes()
print(json.dumps(bench.ffn_bsgs_bench(torch, chain, special, args), indent=1))
