# Why are the first steps of a reverse launch slow?  ncu --set full of rev_tile at 2 and 25 steps per launch.
set -x
for cr in 2 25; do
  LDBP_REV_MAX_STEPS=$cr python scripts/prof_target.py C3 > gpurun_out/pt_c3_cr$cr.log 2>&1 && \
  LDBP_REV_MAX_STEPS=$cr ncu --set full --clock-control none --import-source on -k regex:rev_tile -s 4 -c 1 -o gpurun_out/prof_c3_rev_cr$cr -f python scripts/prof_target.py C3 > gpurun_out/ncu_c3_cr$cr.log 2>&1
  echo rc=$?
  ncu -i gpurun_out/prof_c3_rev_cr$cr.ncu-rep --page source --csv --print-source sass > gpurun_out/src_cr$cr.csv 2>/dev/null
  python scripts/ncu_source_mix.py gpurun_out/src_cr$cr.csv > gpurun_out/mix_cr$cr.txt 2>&1
  ncu -i gpurun_out/prof_c3_rev_cr$cr.ncu-rep --page raw --csv > gpurun_out/raw_cr$cr.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
