# two ranks on one GPU over gloo: the multi-GPU bench path end to end (timing meaningless)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --points 4000000 --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo rc=$?; tail -3 gpurun_out/bench_2rank.err; cut -c1-400 gpurun_out/bench_2rank.json
timeout 900 python -m pytest tests/test_dist_gpu.py -q -m gpu > gpurun_out/dist.log 2>&1; tail -2 gpurun_out/dist.log
