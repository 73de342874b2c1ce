#!/bin/bash
# ncu evidence for the BSGS linear transform (config 3 W1, one matvec after a
# warm-up): per-launch time and DRAM bytes (tools/prof.py ffn exits 0 first).
set -e
python tools/prof.py ffn > gpurun_out/ffn_plain2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ffn_dram.csv python tools/prof.py ffn > gpurun_out/ncu_ffn_dram.log 2>&1
