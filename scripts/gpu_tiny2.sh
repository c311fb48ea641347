set -x
timeout 600 python scripts/tiny_sweep.py
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/tiny_tests.log 2>&1; echo tests_exit=$?
tail -3 gpurun_out/tiny_tests.log
