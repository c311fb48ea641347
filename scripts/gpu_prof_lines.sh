# CUDA-line view of the reverse kernel (C3 and C5 slices): where the once-per-CTA instructions come from
set -x
for c in C3 C5; do
  b=""; [ $c = C5 ] && b=1024
  PROF_B=$b python scripts/prof_target.py $c > /dev/null 2>&1 && \
  PROF_B=$b ncu --set full --clock-control none --import-source on -k regex:rev_tile -s 2 -c 1 -o gpurun_out/prof_${c}_rev -f python scripts/prof_target.py $c > gpurun_out/ncu_${c}_rev.log 2>&1
  ncu -i gpurun_out/prof_${c}_rev.ncu-rep --page source --csv --print-source cuda > gpurun_out/cuda_${c}.csv 2>/dev/null
  ncu -i gpurun_out/prof_${c}_rev.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${c}.csv 2>/dev/null
  python scripts/ncu_cuda_lines.py gpurun_out/cuda_${c}.csv 70 > gpurun_out/lines_${c}.txt 2>&1
  python scripts/ncu_source_mix.py gpurun_out/sass_${c}.csv > gpurun_out/mix_${c}.txt 2>&1
  head -c 3000000 gpurun_out/cuda_${c}.csv > gpurun_out/cuda_${c}_head.csv
  rm -f gpurun_out/sass_${c}.csv gpurun_out/cuda_${c}.csv
done
rm -f gpurun_out/*.ncu-rep
