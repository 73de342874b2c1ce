# tensor-core MAC: parity tests (bounded: a bad descriptor can hang an mbarrier wait) then the probe
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider > gpurun_out/tc_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/tc_tests.log
tail -30 gpurun_out/tc_tests.log
if grep -q "passed" gpurun_out/tc_tests.log && ! grep -q "failed" gpurun_out/tc_tests.log; then
  timeout 300 python tools/mac_tc_probe.py 1 2 4 8 16 > gpurun_out/tc_probe.json 2> gpurun_out/tc_probe.err
  PROBE_SHAPE=w2 timeout 300 python tools/mac_tc_probe.py 1 4 8 > gpurun_out/tc_probe_w2.json 2>> gpurun_out/tc_probe.err
  cat gpurun_out/tc_probe.json gpurun_out/tc_probe_w2.json
fi
