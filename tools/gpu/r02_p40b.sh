timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_p40.py tests/test_gpu_linalg_oracle.py 2>&1 | tail -3
python tools/p40_probe.py > gpurun_out/p40_probe.json 2>&1
for E in 1 0; do
  HX_MAC_P40=$E timeout 900 python tools/ffn_timing.py --only ffn_w1 ffn_w2 ffn_w1_stacked > gpurun_out/p40_ffn_$E.json 2> gpurun_out/p40_ffn_$E.err
done
HX_MAC_P40=1 timeout 600 python tools/config5_timing.py > gpurun_out/p40_c5_1.json 2> gpurun_out/p40_c5_1.err
cat gpurun_out/p40_probe.json; grep -h "ms_per" gpurun_out/p40_ffn_*.json gpurun_out/p40_c5_1.json
