#!/bin/bash
# Per-kernel breakdown of one 256-ciphertext key switch + a full capture of
# the fused ROW/inner-product kernel (run on the GPU box via gpurun; one GPU).
# Usage: tools/prof_ks.sh TAG
set -e
TAG=${1:-ks}
python tools/prof.py ks 256 > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/prof.py ks 256 > /dev/null 2>&1
python tools/ks_breakdown.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_breakdown.txt
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-row_inner|modup_col}" -s ${KSKIP:-2} -c ${KCOUNT:-2} \
    -o /tmp/${TAG}_full -f python tools/prof.py ks 64 > gpurun_out/${TAG}_full.log 2>&1
ncu -i /tmp/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv
ncu -i /tmp/${TAG}_full.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_sass.csv && gzip -c /tmp/${TAG}_sass.csv > gpurun_out/${TAG}_sass.csv.gz
