# round-2 final measurement: default bench (all extras), then the launch list of the headline step
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_final.csv $B > /dev/null 2>&1
echo ncu_rc=$?
