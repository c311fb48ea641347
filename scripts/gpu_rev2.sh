set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$?
tail -15 gpurun_out/gputests.log
LDBP_REV2=1 timeout 300 python scripts/quick_bench.py C3 > gpurun_out/qb.log 2>&1 && cat gpurun_out/qb.log && LDBP_REV2=1 ncu --set full --clock-control none --import-source on -k regex:rev2 -s 2 -c 1 -o gpurun_out/prof_c3_rev2 -f python scripts/prof_target.py C3 > gpurun_out/ncu_c3.log 2>&1
echo ncu=$?
