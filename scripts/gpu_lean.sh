for v in base ob14 lean14 ob14 lean14; do
  if [ "$v" = base ]; then lib=paper_2010_14258_b200/libldbp.so; else lib=build/variants/$v/libldbp.so; fi
  echo "=== $v"; LDBP_LIB=$lib timeout 300 python scripts/quick_bench.py C3 C5 2>&1 | grep -v Warn | grep -v "kind 3"
done
echo "=== parity (lean14)"; LDBP_LIB=build/variants/lean14/libldbp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -q -x -k "loss_grad or backward or determinism or timed or repeated" 2>&1 | tail -3
