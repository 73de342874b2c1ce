#!/bin/bash
# Profiles committed under profiles/ (run on the GPU box via gpurun; one GPU).
# 1. the bench command exits 0 without ncu, 2. its launch list (timings only),
# 3. one --set full capture per top kernel of a 64-ciphertext key switch.
set -e
python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"modup_col|ks_inner_f64|combine_kernel|moddown_bconv" -s 4 -c 4 \
    -o gpurun_out/prof_ks_full -f python tools/prof.py ks 64 > gpurun_out/ncu_ks_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ntt_pass -s 0 -c 8 \
    -o gpurun_out/prof_ntt_full -f python tools/prof.py ntt 64 > gpurun_out/ncu_ntt_full.log 2>&1
