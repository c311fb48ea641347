set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py tests/test_gpu_fullsize.py tests/test_gpu_rx.py tests/test_pruning.py -x -q 2>&1 | tail -3
bash scripts/gpu_variants.sh "C3 C5" base nobulk
