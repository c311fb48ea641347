set -x
export LDBP_REV2=0 PROF_B=1024
python scripts/prof_target.py C5 > gpurun_out/pt_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rev_tile -s 1 -c 1 -o gpurun_out/prof_c5_rev -f python scripts/prof_target.py C5 > gpurun_out/ncu_c5.log 2>&1
echo rc=$?
