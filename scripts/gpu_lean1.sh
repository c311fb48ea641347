for v in base lean1 base lean1 base lean1; do
  if [ "$v" = base ]; then lib=paper_2010_14258_b200/libldbp.so; else lib=build/variants/$v/libldbp.so; fi
  echo "=== $v"; LDBP_LIB=$lib timeout 300 python scripts/quick_bench.py C5 2>&1 | grep -v Warn | grep -v "kind 3"
done
