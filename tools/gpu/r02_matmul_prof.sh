# launch list of the config-4 ct-ct matmul (d = 128, one head) at 3 and 4 limbs
for L in 3 4; do
cat > /tmp/mm_$L.py <<EOF
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
chain, special = bench.primes()
print(bench.matmul_bench(torch, chain, special, n_q=$L, iters=1, heads=0))
EOF
python /tmp/mm_$L.py > gpurun_out/r02_mm_l$L.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_mm_l$L.csv python /tmp/mm_$L.py > /dev/null 2>&1
echo rc=$?; tail -1 gpurun_out/r02_mm_l$L.log | cut -c1-300
done
