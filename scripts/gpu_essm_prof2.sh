set -x
python scripts/essm_bench.py 2>&1 | tail -4
python scripts/essm_prof_target.py > gpurun_out/pt_essm.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:essm_ -s 0 -c 4 -o gpurun_out/prof_essm -f python scripts/essm_prof_target.py > gpurun_out/ncu_essm.log 2>&1
echo ncu=$?
python scripts/kernel_metrics.py gpurun_out/prof_essm.ncu-rep
