# round evidence on one B200: full GPU suite, smoke, sanitizers, default bench -> gpurun_out/
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
timeout 2400 python -m pytest tests -m gpu -q -rs --timeout 1500 > gpurun_out/gpu_tests.log 2>&1; tail -8 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --stages > gpurun_out/bench_cluster2B_color_filter.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
[ -n "$SANITIZE" ] && bash scripts/sanitize.sh
true
