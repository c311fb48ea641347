set -x
./scripts/microbench > gpurun_out/microbench.txt 2>&1
python scripts/prof_target.py C2 > gpurun_out/pt_c2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fwd_tile -s 1 -c 1 -o gpurun_out/prof_c2_fwd -f python scripts/prof_target.py C2 > gpurun_out/ncu_c2.log 2>&1
python scripts/prof_target.py C3 > gpurun_out/pt_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:bwd_segment -s 10 -c 1 -o gpurun_out/prof_c3_bwd -f python scripts/prof_target.py C3 > gpurun_out/ncu_c3.log 2>&1
python bench.py --steps 2 --warmup 3 --no-extra --no-cpu > gpurun_out/b_small.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo done
