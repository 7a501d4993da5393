# quick B200 check of a change: focused GPU tests + bench stage times -> gpurun_out/
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
timeout 1800 python -m pytest tests -m gpu -q -x -rs --timeout 1200 ${TESTS:-} > gpurun_out/gpu_tests.log 2>&1; tail -8 gpurun_out/gpu_tests.log
for c in ${CONFIGS:-cluster2B}; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --stages --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/bq_$c.json 2> gpurun_out/bq_$c.err; tail -2 gpurun_out/bq_$c.err
done
