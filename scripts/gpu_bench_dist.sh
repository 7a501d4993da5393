# N=2 bench code path on ONE GPU (gloo collectives, two ranks sharing cuda:0)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --backend gloo --steps 2 --warmup 3 --points 4000000 --no-cpu-baseline > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err; tail -5 gpurun_out/bench_dist.err; cat gpurun_out/bench_dist.json
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
