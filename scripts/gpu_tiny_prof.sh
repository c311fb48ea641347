set -x
python scripts/tiny_prof_target.py > gpurun_out/pt_tiny.log 2>&1 && ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:tiny -s 4 -c 1 -o gpurun_out/prof_tiny -f python scripts/tiny_prof_target.py > gpurun_out/ncu_tiny.log 2>&1
echo ncu=$?
