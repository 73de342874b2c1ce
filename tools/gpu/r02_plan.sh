# cost-tuned BSGS split: parity of explicit plans vs the oracle, then W1 at n1 = 32 (SPEC) / 64 (for_cost) / 128
python -m pytest tests/test_gpu_linalg_oracle.py -q -x -k "explicit_plan or config1_bsgs" 2>&1 | tail -3
python tools/ffn_timing.py --no-w2 --only ffn_w1 ffn_w1_cost_plan > gpurun_out/r02_plan_w1.json 2> gpurun_out/r02_plan_w1.err; echo rc=$?
HX_BENCH_N1=128 python tools/ffn_timing.py --no-w2 --only ffn_w1 > gpurun_out/r02_plan_w1_n128.json 2>> gpurun_out/r02_plan_w1.err; echo rc=$?
HX_BENCH_N1=16 python tools/ffn_timing.py --no-w2 --only ffn_w1_stacked > gpurun_out/r02_plan_w1s_n16.json 2>> gpurun_out/r02_plan_w1.err; echo rc=$?
HX_BENCH_N1=64 python tools/ffn_timing.py --no-w2 --only ffn_w1_stacked > gpurun_out/r02_plan_w1s_n64.json 2>> gpurun_out/r02_plan_w1.err; echo rc=$?
grep -h "ms_per_matvec\|ms_per_token\|\"n1\"\|^ \"ffn" gpurun_out/r02_plan_w1*.json
HX_BENCH_DEVICE=0 HX_BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 \
  > gpurun_out/r02_world2.json 2> gpurun_out/r02_world2.err
echo world2_rc=$?; tail -c 1500 gpurun_out/r02_world2.json; grep -v "^$" gpurun_out/r02_world2.err | tail -5
