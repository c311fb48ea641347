# e2e A/B: the step on a high-priority stream (default) vs the default stream
for p in 0 1 0 1; do echo "=== LDBP_BENCH_E2E_PRIO=$p"; LDBP_BENCH_E2E_PRIO=$p timeout 300 python bench.py --no-extra --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
