# TC MAC after the builder lane reorder: parity tests, W1 / W2 probes, one ncu capture (bank conflicts)
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tc.py tests/test_gpu_linalg_oracle.py 2>&1 | tail -2
python tools/mac_tc_probe.py 1 2 4 8 16 > gpurun_out/tc2_w1.json 2> gpurun_out/tc2_w1.err
PROBE_SHAPE=w2 python tools/mac_tc_probe.py 1 4 8 > gpurun_out/tc2_w2.json 2> gpurun_out/tc2_w2.err
PROBE_REPS=1 ncu --set full --clock-control none --import-source on -k regex:bsgs_mac_tc -s 2 -c 1 -o gpurun_out/r02_tc2_t8 python tools/mac_tc_probe.py 8 > gpurun_out/tc2_ncu8.log 2>&1
echo rc=$?
