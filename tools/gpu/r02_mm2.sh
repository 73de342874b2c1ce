# low-dnum ks_inner instances: parity subset, then the config-4 matmul at 3 / 4 limbs
python -m pytest tests/test_gpu_linalg_oracle.py tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -x -k "matmul or keyswitch or rotate or inner or relin" 2>&1 | tail -3
for L in 3 4; do
cat > /tmp/mm_$L.py <<EOF
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
chain, special = bench.primes()
print(bench.matmul_bench(torch, chain, special, n_q=$L, iters=2, heads=12))
EOF
python /tmp/mm_$L.py 2>&1 | tail -1 | cut -c1-600
done
