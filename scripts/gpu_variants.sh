# A/B timing of library variants: bash scripts/gpu_variants.sh "C3 C5" base nw4 nw2 ...
cfgs="$1"; shift
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2010_14258_b200/libldbp.so; else lib=build/variants/$v/libldbp.so; fi
  echo "=== $v"
  LDBP_LIB=$lib timeout 300 python scripts/quick_bench.py $cfgs 2>&1 | grep -v Warn
done
