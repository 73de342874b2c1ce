# P40 packed MAC: parity, then FFN / config-5 timings with and without it
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_p40.py tests/test_gpu_linalg_oracle.py tests/test_gpu_helix.py 2>&1 | tail -3
for E in 1 0; do
  HX_MAC_P40=$E timeout 600 python tools/ffn_timing.py --only ffn_w1 ffn_w2 ffn_w1_stacked > gpurun_out/p40_ffn_$E.json 2> gpurun_out/p40_ffn_$E.err
  HX_MAC_P40=$E timeout 600 python tools/config5_timing.py > gpurun_out/p40_c5_$E.json 2> gpurun_out/p40_c5_$E.err
done
grep -h "ms_per_matvec" gpurun_out/p40_*.json | head -20
PROBE_REPS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p40_launches.csv python bench.py --steps 1 --warmup 3 --no-extras --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bsgs_mac_p40 -c 1 -o gpurun_out/r02_p40 python bench.py --steps 1 --warmup 3 --no-extras --no-cpu > /dev/null 2>&1
echo rc=$?
