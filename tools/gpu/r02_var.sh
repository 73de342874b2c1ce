# run-to-run variance of the token-batched extras: allocation trace on
for i in 1 2 3; do
HX_ALLOC_TRACE=1 python tools/ffn_timing.py --no-w2 --only ffn_w1_stacked 2> gpurun_out/r02_var_$i.err | grep -h "ms_per"
grep -c "trim" gpurun_out/r02_var_$i.err; grep "regrown" gpurun_out/r02_var_$i.err | tail -3
done
