# launch list of one FFN W1 matvec (T = 1) on the cost-tuned split
cat > /tmp/w1.py <<EOF
import sys, os, argparse
sys.path.insert(0, os.getcwd())
import torch, bench
chain, special = bench.primes()
args = argparse.Namespace(no_w2=True, only=["ffn_w1_cost_plan"], verbose=False)
print(bench.ffn_bsgs_bench(torch, chain, special, args, iters=1, tokens=0))
EOF
python /tmp/w1.py > gpurun_out/r02_w1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_w1_launches.csv python /tmp/w1.py > /dev/null 2>&1
echo rc=$?; tail -1 gpurun_out/r02_w1_plain.log | cut -c1-300
