# bench.py --gpus 2 orchestration on ONE GPU (2 ranks, gloo collectives) -> gpurun_out/bench_2rank_*.json
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in terrain20M scene500M; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --config $c --backend gloo --points ${PTS:-0} > gpurun_out/bench_2rank_$c.json 2> gpurun_out/bench_2rank_$c.err
tail -3 gpurun_out/bench_2rank_$c.err; head -c 600 gpurun_out/bench_2rank_$c.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29534 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --config terrain20M > gpurun_out/bench_2rank_reference.json 2>> gpurun_out/bench_2rank_terrain20M.err
head -c 400 gpurun_out/bench_2rank_reference.json
