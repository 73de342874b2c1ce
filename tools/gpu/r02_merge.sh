# merged-block P40 MAC: parity, then W1 on the cost-tuned split with and without the merge
python -m pytest tests/test_gpu_linalg_oracle.py tests/test_gpu_p40.py tests/test_gpu_helix.py -q -x 2>&1 | tail -2
for m in 0 1; do echo "HX_P40_MERGE=$m"; HX_P40_MERGE=$m python tools/ffn_timing.py --no-w2 --only ffn_w1_cost_plan 2>/dev/null | grep -h "ms_per_matvec\|max_abs"; done
python tools/ffn_timing.py --only ffn_w2 2>/dev/null | grep -h "ms_per_matvec"
python tools/p40_probe.py 2>&1 | tail -6
