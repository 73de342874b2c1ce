cat > /tmp/mm.py <<EOF
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
chain, special = bench.primes()
r = bench.matmul_bench(torch, chain, special, n_q=3, iters=2, heads=0); print(r["ms_per_matmul"], r["ms_per_iteration"])
c47, s47 = bench.primes(fp64_specials=True)
for _ in range(2):
    r = bench.matmul_bench(torch, c47, s47, heads=0); print(r["ms_per_matmul"], r["ms_per_iteration"])
EOF
python /tmp/mm.py 2>&1 | tail -4
