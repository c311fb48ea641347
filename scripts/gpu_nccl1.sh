# One-rank NCCL exchange on hardware: the DP trainer test and the C3 step with the forced all-reduce.
set -x
timeout 600 python -m pytest tests/test_gpu_dp_nccl.py -q > gpurun_out/nccl_test.log 2>&1; echo test_exit=$?
tail -5 gpurun_out/nccl_test.log
timeout 600 python bench.py --no-extra --no-cpu > gpurun_out/bench_c3_plain.json 2> gpurun_out/bench_c3_plain.err; echo plain_exit=$?
timeout 600 python bench.py --no-extra --no-cpu --force-collective > gpurun_out/bench_c3_nccl1.json 2> gpurun_out/bench_c3_nccl1.err; echo nccl_exit=$?
grep -i "NCCL INFO" gpurun_out/bench_c3_nccl1.err | head -20
python - <<'P'
import json
for f in ("bench_c3_plain", "bench_c3_nccl1"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, d["value"], d["ms_per_step"], d["dist_backend"], d["gpu_launches"], d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e)
P
