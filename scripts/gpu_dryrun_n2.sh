# The bench's N = 2 path end to end as a gloo dry run on one GPU (both ranks share the device:
# a functional check of sharding, the training all-reduce, e2e and max-over-ranks timing; not a scaling number)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --config C3 --no-extra --no-cpu --dist-backend gloo > gpurun_out/dry_c3_n2.json 2> gpurun_out/dry_c3_n2.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --config C4 --no-extra --no-cpu --no-e2e --dist-backend gloo > gpurun_out/dry_c4_n2.json 2> gpurun_out/dry_c4_n2.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/dry_ref_n2.json 2> gpurun_out/dry_ref_n2.err; echo rc=$?
tail -c 600 gpurun_out/dry_c3_n2.err
