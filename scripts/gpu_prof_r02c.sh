# ncu --set full captures of the C3 training-step kernels and the C2 forward (round 2, third session).
set -x
python scripts/prof_target.py C3 > gpurun_out/pt_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rev_tile|fwd_store" -s 3 -c 2 \
  -o gpurun_out/r02c_c3 -f python scripts/prof_target.py C3 > gpurun_out/ncu_c3.log 2>&1; echo c3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_tile -s 1 -c 1 \
  -o gpurun_out/r02c_c2 -f python scripts/prof_target.py C2 > gpurun_out/ncu_c2.log 2>&1; echo c2=$?
python scripts/kernel_metrics.py gpurun_out/r02c_c3.ncu-rep gpurun_out/r02c_c2.ncu-rep > gpurun_out/r02c_kernel_metrics.txt 2>&1
cat gpurun_out/r02c_kernel_metrics.txt
