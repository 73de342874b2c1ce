# T = 1 tensor-core MAC threshold: W1 on the cost-tuned split (3 x 16 = 48 rows, n1 = 64)
for R in 96 48; do
echo "HX_TC_MIN_ROWS=$R"
HX_TC_MIN_ROWS=$R python tools/ffn_timing.py --no-w2 --only ffn_w1_cost_plan 2>/dev/null | grep -h "ms_per\|max_abs"
done
