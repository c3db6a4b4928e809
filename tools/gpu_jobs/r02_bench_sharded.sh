# Validation of bench.py's sharded path (N > 1) on one GPU: two gloo ranks sharing it, config 3.
MLE_BENCH_CONFIG=config3 MLE_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_sharded_validation.json 2> gpurun_out/bench_sharded_validation.err; echo rc=$?
tail -c 1500 gpurun_out/bench_sharded_validation.json; tail -5 gpurun_out/bench_sharded_validation.err
