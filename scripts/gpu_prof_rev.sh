set -x
python scripts/prof_target.py C3 > gpurun_out/pt_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rev_tile -s 2 -c 1 -o gpurun_out/prof_c3_rev -f python scripts/prof_target.py C3 > gpurun_out/ncu_c3.log 2>&1
echo rc=$?
