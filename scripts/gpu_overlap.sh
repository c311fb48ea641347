set -x
for k in 1 2 4 8; do echo "== OVERLAP=$k"; LDBP_OVERLAP=$k timeout 300 python scripts/quick_bench.py C3 C5 2>&1 | grep -v Warn | grep -v "kind"; done
timeout 900 python -m pytest tests/test_gpu_timed_path.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
