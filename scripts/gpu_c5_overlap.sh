for k in 0 2 3; do echo "=== LDBP_OVERLAP=$k"; LDBP_OVERLAP=$k timeout 300 python scripts/quick_bench.py C5 2>&1 | grep -v Warn | grep "wall"; done
