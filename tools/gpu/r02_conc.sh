timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_concurrency.py tests/test_gpu_helix.py tests/test_gpu_acceptance.py tests/test_gpu_linalg_oracle.py tests/test_gpu_cpp_api.py tests/test_gpu_shard_mp.py tests/test_gpu_cli.py 2>&1 | tail -4
timeout 600 python tools/ffn_timing.py --only ffn_w1 ffn_w2 > gpurun_out/ffn_conc.json 2> gpurun_out/ffn_conc.err; grep -h "ms_per" gpurun_out/ffn_conc.json
timeout 600 python tools/matmul_timing.py 2>&1 | tail -1 | cut -c1-300
