set -x
python scripts/essm_bench.py 2>&1 | tail -4
python scripts/essm_prof_target.py > gpurun_out/pt_essm.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:essm_bwd -s 1 -c 1 -o gpurun_out/prof_essm_bwd -f python scripts/essm_prof_target.py > gpurun_out/ncu_essm.log 2>&1
echo ncu=$?
