# ncu full capture of the one-element key inner product (63 hoisted baby steps of one W1 matvec)
cat > /tmp/w1.py <<EOF
import sys, os, argparse
sys.path.insert(0, os.getcwd())
import torch, bench
chain, special = bench.primes()
args = argparse.Namespace(no_w2=True, only=["ffn_w1_cost_plan"], verbose=False)
print(bench.ffn_bsgs_bench(torch, chain, special, args, iters=1, tokens=0))
EOF
python /tmp/w1.py > gpurun_out/r02_w1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ks_inner_f64_one -s 2 -c 1 -o gpurun_out/r02_inner_one python /tmp/w1.py > /dev/null 2>&1
echo rc=$?
