timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_linalg_oracle.py tests/test_gpu_helix.py 2>&1 | tail -2
timeout 600 python tools/ffn_timing.py --only ffn_w1 ffn_w2 > gpurun_out/ffn_s.json 2> gpurun_out/ffn_s.err; grep -h "ms_per" gpurun_out/ffn_s.json
timeout 900 python tools/matmul_timing.py 2>&1 | tail -1 | cut -c1-400
