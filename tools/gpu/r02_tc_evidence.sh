# round 2: tensor-core vs CUDA-core BSGS MAC (W1 / W2 shapes), ncu SASS evidence of the
# tcgen05 MAC, and a source-level ncu capture of the ModUp kernel for stall attribution
python tools/mac_tc_probe.py 1 2 4 8 16 > gpurun_out/tc_w1.json 2> gpurun_out/tc_w1.err
PROBE_SHAPE=w2 python tools/mac_tc_probe.py 1 4 8 > gpurun_out/tc_w2.json 2> gpurun_out/tc_w2.err
export PROBE_REPS=1
ncu --set full --clock-control none --import-source on -k regex:bsgs_mac_tc -s 2 -c 1 -o gpurun_out/r02_tc_t8 python tools/mac_tc_probe.py 8 > gpurun_out/tc_ncu8.log 2>&1
cuobjdump -sass paper_2512_11135_b200/libhx_b200.so | grep -E "UTC|UBLKCP|UTMA|LDTM" | sort | uniq -c | sort -rn | head -20 > gpurun_out/tc_sass_ops.txt
B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:modup_col -s 4 -c 1 -o gpurun_out/r02_modup_src $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ntt_pass_kernel -s 20 -c 4 -o gpurun_out/r02_ntt_src $B > /dev/null 2>&1
echo rc=$?
ls -la gpurun_out
