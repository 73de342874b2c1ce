# two rows per step in the n1 = 64 packed MAC: parity, A/B
HX_P40_RPS=2 python -m pytest tests/test_gpu_p40.py tests/test_gpu_linalg_oracle.py -q -x -k "p40 or explicit_plan" 2>&1 | tail -2
for r in 1 2; do echo "HX_P40_RPS=$r"; HX_P40_RPS=$r python tools/p40_probe.py 2>/dev/null | grep -h "p40_ms\|p40_GBps"; done
for r in 1 2; do echo "HX_P40_RPS=$r"; HX_P40_RPS=$r python tools/ffn_timing.py --only ffn_w1_cost_plan ffn_w2 2>/dev/null | grep -h "ms_per_matvec"; done
