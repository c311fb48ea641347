set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py tests/test_pruning.py -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$?
tail -25 gpurun_out/gputests.log
for v in 0 1; do LDBP_REV3=$v timeout 300 python scripts/quick_bench.py C3 C2 2>&1 | grep -v Warn; done
