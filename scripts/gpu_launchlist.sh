timeout 300 python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_exit=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_exit=$?
