for v in base onebody base onebody; do
  if [ "$v" = base ]; then lib=paper_2010_14258_b200/libldbp.so; else lib=build/variants/$v/libldbp.so; fi
  echo "=== $v"; LDBP_LIB=$lib timeout 300 python scripts/quick_bench.py C3 2>&1 | grep -v Warn
done
echo "=== parity (onebody)"; LDBP_LIB=build/variants/onebody/libldbp.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "loss_grad or backward or determinism" 2>&1 | tail -3
python scripts/prof_target.py C3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rev_tile -s 2 -c 1 -o gpurun_out/prof_c3_rev_cr25 -f python scripts/prof_target.py C3 > gpurun_out/ncu_c3_cr25.log 2>&1
ncu -i gpurun_out/prof_c3_rev_cr25.ncu-rep --page source --csv --print-source sass > gpurun_out/src_cr25.csv 2>/dev/null
python scripts/ncu_source_mix.py gpurun_out/src_cr25.csv > gpurun_out/mix_cr25.txt 2>&1
ncu -i gpurun_out/prof_c3_rev_cr25.ncu-rep --page raw --csv > gpurun_out/raw_cr25.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
grep -n "stall_" gpurun_out/mix_cr25.txt | head -6
