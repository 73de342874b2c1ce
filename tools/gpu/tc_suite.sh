timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_linalg_oracle.py -x -q -p no:cacheprovider > gpurun_out/tc_suite.log 2>&1; echo rc=$? >> gpurun_out/tc_suite.log
tail -5 gpurun_out/tc_suite.log
