# C3 / C5 training step vs steps per reverse launch (runtime knob LDBP_REV_MAX_STEPS)
for s in 10 13 17 25 50; do echo "=== LDBP_REV_MAX_STEPS=$s"; LDBP_REV_MAX_STEPS=$s timeout 300 python scripts/quick_bench.py C3 2>&1 | grep -v Warn; done
for s in 9 13 25; do echo "=== C5 LDBP_REV_MAX_STEPS=$s"; LDBP_REV_MAX_STEPS=$s timeout 300 python scripts/quick_bench.py C5 2>&1 | grep -v Warn; done
