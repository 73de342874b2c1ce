# W1 at n1 = 32 (SPEC) / 64 (for_cost) / 128, one token and 128 tokens
python tools/ffn_timing.py --no-w2 --only ffn_w1 ffn_w1_cost_plan > gpurun_out/r02_plan_w1.json 2> gpurun_out/r02_plan_w1.err; echo rc=$?
HX_BENCH_N1=128 python tools/ffn_timing.py --no-w2 --only ffn_w1 > gpurun_out/r02_plan_w1_n128.json 2>> gpurun_out/r02_plan_w1.err; echo rc=$?
HX_BENCH_N1=64 python tools/ffn_timing.py --no-w2 --only ffn_w1_pruned90 > gpurun_out/r02_plan_w1p_n64.json 2>> gpurun_out/r02_plan_w1.err; echo rc=$?
grep -h "ms_per_matvec\|ms_per_token\|\"n1\"\|^ \"ffn\|rotations\|chunk" gpurun_out/r02_plan_w1.json gpurun_out/r02_plan_w1_n128.json gpurun_out/r02_plan_w1p_n64.json
