set -x


LDBP_REV3=1 timeout 300 python scripts/quick_bench.py C3 > gpurun_out/qb.log 2>&1 && cat gpurun_out/qb.log && LDBP_REV3=1 ncu --set full --clock-control none --import-source on -k regex:rev3 -s 2 -c 1 -o gpurun_out/prof_c3_rev3 -f python scripts/prof_target.py C3 > gpurun_out/ncu_c3.log 2>&1
echo ncu=$?
