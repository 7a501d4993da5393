# one B200 evidence pass -> gpurun_out/ : GPU tests (new large-config parity first), smoke, bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1500 ${TESTS:-} > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --stages > gpurun_out/bench_cluster2B_color_filter.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
