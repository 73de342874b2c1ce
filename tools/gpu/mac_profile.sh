# BSGS MAC alone (FFN W1 block shape): launch list at T = 1 / 16 and one ncu full capture of the FP64 MAC at T = 16
export PROBE_REPS=1
python tools/mac_tokens_probe.py 1 16 > gpurun_out/mac_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mac_launches.csv python tools/mac_tokens_probe.py 1 16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bsgs_mac_f64 -s 3 -c 1 -o gpurun_out/mac_f64_t16 python tools/mac_tokens_probe.py 16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bsgs_mac_f64 -s 3 -c 1 -o gpurun_out/mac_f64_t1 python tools/mac_tokens_probe.py 1 > /dev/null 2>&1
echo done
