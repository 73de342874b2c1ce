# inner-product grids with (key, slice) fastest: parity, then key-switch / hoisted / FFN timings
python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_edge.py -q -x 2>&1 | tail -2
for op in rotate relin hoisted; do python tools/ks_time.py 256 $op 2>&1 | tail -1; done
python tools/ffn_timing.py --only ffn_w1 ffn_w1_cost_plan ffn_w1_stacked ffn_w2 2>/dev/null | grep -h "ms_per_matvec\|ms_per_token\|^ \"ffn"
