# round-2 check of bench.py's multi-rank glue on a single-GPU box: two ranks on
# GPU 0 over gloo (HX_BENCH_DEVICE / HX_BENCH_DIST_BACKEND).  Not a reported
# number -- the ranks share one device.  Then the launch list and full captures
# of the headline step at HEAD.
HX_BENCH_DEVICE=0 HX_BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 \
  > gpurun_out/r02_world2.json 2> gpurun_out/r02_world2.err
echo world2_rc=$?; tail -c 1200 gpurun_out/r02_world2.json; tail -5 gpurun_out/r02_world2.err
B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_head.csv $B > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:modup_col -s 4 -c 1 -o gpurun_out/r02_modup_col_head $B > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ks_row_inner -s 4 -c 1 -o gpurun_out/r02_rowinner_head $B > /dev/null 2>&1
echo ncu_rc=$?
