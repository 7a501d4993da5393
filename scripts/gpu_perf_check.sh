# focused parity (extension / 2-pass distribute / large configs) + stage times -> gpurun_out/
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_large.py -m gpu -q -x -rs --timeout 1200 -k "${KSEL:-many_leaves or two_pass or cluster or stadium or scene or initial6 or depth_limit}" > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
for c in ${CONFIGS:-cluster2B terrain20M}; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --stages --no-cpu-baseline --no-e2e > gpurun_out/bq_$c.json 2> gpurun_out/bq_$c.err; tail -1 gpurun_out/bq_$c.err
python -c "import json; d=json.loads(open('gpurun_out/bq_$c.json').read()); print('$c', d['value']/1e9, d['ms_per_step'])"
done
