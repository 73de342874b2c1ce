HX_ALLOC_TRACE=1 python tools/ffn_timing.py --no-w2 2> gpurun_out/r02_var_seq.err | grep -h "ms_per\|^ \"ffn"
grep -n "trim\|regrown" gpurun_out/r02_var_seq.err | tail -40
