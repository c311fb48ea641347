for v in base noob23 base noob23; do
  if [ "$v" = base ]; then lib=paper_2010_14258_b200/libldbp.so; else lib=build/variants/$v/libldbp.so; fi
  echo "=== $v"; LDBP_LIB=$lib timeout 300 python scripts/kh_train_bench.py 5 7 2>&1 | grep "T="
done
