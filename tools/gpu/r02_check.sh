# round-2 re-entry check: full GPU test suite, smoke, and a default bench run
set -o pipefail
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/gputests.log; tail -2 gpurun_out/smoke.log
