# C2 forward vs CTA size (runtime knob LDBP_FWD_THREADS): smaller tiles = more waves, more halo
for t in 32 64 96 128; do echo "=== LDBP_FWD_THREADS=$t"; LDBP_FWD_THREADS=$t timeout 300 python scripts/quick_bench.py C2 2>&1 | grep -v Warn; done
