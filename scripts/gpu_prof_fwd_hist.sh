set -x
run() { # name cfg kernel-regex skip env
  PROF_FWD=$5 python scripts/prof_target.py $2 > /dev/null 2>&1
  PROF_FWD=$5 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o gpurun_out/p_$1 -f python scripts/prof_target.py $2 > gpurun_out/ncu_$1.log 2>&1
  ncu -i gpurun_out/p_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/s_$1.csv 2>/dev/null
  ncu -i gpurun_out/p_$1.ncu-rep --page raw --csv > gpurun_out/r_$1.csv 2>/dev/null
  W=$(python - <<P
import csv
rows=list(csv.reader(open("gpurun_out/r_$1.csv"))); h=rows[0]; r=rows[-1]
g=float(r[h.index("launch__grid_size")]); b=float(r[h.index("launch__block_size")]); print(int(g*b/32))
P
)
  python scripts/ncu_exec_hist.py gpurun_out/s_$1.csv $W > gpurun_out/hist_$1.txt 2>&1
  python scripts/ncu_source_mix.py gpurun_out/s_$1.csv > gpurun_out/mix_$1.txt 2>&1
  python - <<P >> gpurun_out/hist_$1.txt
import csv
rows=list(csv.reader(open("gpurun_out/r_$1.csv"))); h=rows[0]; r=rows[-1]
for k in ("gpu__time_duration.sum","sm__icc_request_hit_rate.pct","smsp__issue_active.avg.pct_of_peak_sustained_active","sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active","launch__grid_size","launch__block_size","launch__registers_per_thread"):
    print(k, r[h.index(k)])
P
  rm -f gpurun_out/s_$1.csv gpurun_out/p_$1.ncu-rep gpurun_out/r_$1.csv
}
run fwdstore_C3 C3 fwd_store 1 ""
run fwd_C2 C2 fwd_tile 1 ""
run fwd_C4 C4 fwd_tile 1 ""
run rev_C5 C5 rev_tile 1 ""
