# ncu full capture of the packed MAC at n1 = n2 = 64 (KPT = 8), after the plain run exited 0
python tools/p40_probe.py > gpurun_out/p40_plain.json 2> gpurun_out/p40_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:bsgs_mac_p40 -s 9 -c 1 -o gpurun_out/r02_p40_n64 python tools/p40_probe.py > /dev/null 2>&1
echo rc=$?; cat gpurun_out/p40_plain.json | tr -d '\n' | cut -c1-400
