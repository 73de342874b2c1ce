export PROBE_REPS=1
ncu --set full --clock-control none --import-source on -k regex:bsgs_mac_tc_kernel -s 2 -c 1 -o gpurun_out/tc_t8 python tools/mac_tc_probe.py 8 > gpurun_out/tc_ncu8.log 2>&1
ls -la gpurun_out/*.ncu-rep
