for s in 1 2 5; do echo "=== LDBP_REV_MAX_STEPS=$s"; LDBP_REV_MAX_STEPS=$s timeout 300 python scripts/quick_bench.py C3 2>&1 | grep -v Warn; done
