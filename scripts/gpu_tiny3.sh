set -x
timeout 600 python scripts/tiny_sweep.py > gpurun_out/tiny_sweep.txt 2>&1; echo sweep_exit=$?
timeout 300 python scripts/c1_graph.py; echo c1_exit=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$?
tail -5 gpurun_out/gputests.log
