# round-2 GPU session: GPU tests, a bench pass, then the ncu launch list + full captures of the top key-switch kernels
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/b4.json 2> gpurun_out/b4.err
B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv $B > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:modup_col -s 4 -c 1 -o gpurun_out/r02_modup_col $B > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ks_row_inner -s 4 -c 1 -o gpurun_out/r02_rowinner $B > /dev/null 2>&1
echo ncu_rc=$?
ls -la gpurun_out/
