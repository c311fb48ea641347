set -x
for m in 1 0; do LDBP_BWD_MODE=$m timeout 300 python scripts/quick_bench.py C5 2>&1 | grep -v Warn; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --config C4 --no-extra --no-cpu --no-e2e --dist-backend gloo > gpurun_out/dry_c4_n2.json 2> gpurun_out/dry_c4_n2.err; echo rc=$?
tail -c 1200 gpurun_out/dry_c4_n2.json; tail -3 gpurun_out/dry_c4_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --config C3 --no-extra --no-cpu --dist-backend gloo > gpurun_out/dry_c3_n2.json 2> gpurun_out/dry_c3_n2.err; echo rc=$?
tail -c 1500 gpurun_out/dry_c3_n2.json; tail -3 gpurun_out/dry_c3_n2.err
