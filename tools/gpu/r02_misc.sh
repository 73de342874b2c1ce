./tools/microbench/fp64lat > gpurun_out/fp64lat.txt 2>&1
timeout 900 python tools/ffn_timing.py --only ffn_w1 ffn_w2 > gpurun_out/ffn_r3.json 2> gpurun_out/ffn_r3.err
cat gpurun_out/fp64lat.txt; grep -h "ms_per" gpurun_out/ffn_r3.json
