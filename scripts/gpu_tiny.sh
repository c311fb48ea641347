# C1 fused one-cluster training step: parity tests, graph latency, launch list.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/tiny_tests.log 2>&1; echo tests_exit=$?
tail -15 gpurun_out/tiny_tests.log
timeout 300 python scripts/c1_graph.py; echo c1_exit=$?
LDBP_TINY=0 timeout 300 python scripts/c1_graph.py; echo c1_seg_exit=$?
timeout 600 python bench.py --config C1 --steps 20 --warmup 3 --no-extra --no-cpu 2> gpurun_out/c1_bench.err | tee gpurun_out/c1_bench.json; echo bench_exit=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tiny --csv --log-file gpurun_out/tiny_launches.csv python bench.py --config C1 --steps 5 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1; echo ncu_exit=$?
grep -c tiny gpurun_out/tiny_launches.csv; tail -3 gpurun_out/tiny_launches.csv
