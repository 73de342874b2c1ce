ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tok8_launches.csv python tools/tokens_chunk_probe.py --once 8 > /dev/null 2>&1
echo rc=$?
