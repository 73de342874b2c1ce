set -e
python tools/prof.py ks 64 > gpurun_out/ks64_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ks64c.csv python tools/prof.py ks 64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"modup_bconv|moddown_bconv|combine_kernel|ks_inner_f64|permute_multi" -s 8 -c 5 -o gpurun_out/prof_ks4 -f python tools/prof.py ks 64 > gpurun_out/ncu_ks4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ntt_pass" -s 16 -c 8 -o gpurun_out/prof_ntt3 -f python tools/prof.py ks 64 > gpurun_out/ncu_ntt3.log 2>&1
