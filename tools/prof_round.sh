#!/bin/bash
# Profiles committed under profiles/ (run on the GPU box via gpurun; one GPU).
# 1. the bench command exits 0 without ncu, 2. its launch list (timings only),
# 3. --set full captures of the key-switch and NTT kernels; the .ncu-rep files
#    stay in /tmp on the box (too large to bring back), their raw / details
#    pages come back as CSV.
set -e
TAG=${1:-prof}
python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > gpurun_out/${TAG}_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"modup_col|ks_row_inner|ks_inner|row_combine" -s 6 -c 6 \
    -o /tmp/${TAG}_ks_full -f python tools/prof.py ks 64 > gpurun_out/${TAG}_ncu_ks_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ntt_pass -s 0 -c 8 \
    -o /tmp/${TAG}_ntt_full -f python tools/prof.py ntt 64 > gpurun_out/${TAG}_ncu_ntt_full.log 2>&1
for r in ks ntt; do
  ncu -i /tmp/${TAG}_${r}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_${r}_full_raw.csv
  ncu -i /tmp/${TAG}_${r}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_${r}_full_details.csv
done
