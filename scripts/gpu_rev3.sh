set -x
for v in 0 1; do LDBP_REV3=$v timeout 300 python scripts/quick_bench.py C3 2>&1 | grep -v Warn; done
LDBP_REV3=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py tests/test_pruning.py -x -q 2>&1 | tail -3
