# Round-2 GPU check: -m gpu tests, smoke, default bench line.
set -x
nproc
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$?
tail -30 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
cat gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench_exit=$?
tail -c 1500 gpurun_out/bench_full.json
tail -5 gpurun_out/bench_full.err
