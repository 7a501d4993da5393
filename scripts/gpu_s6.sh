mkdir -p gpurun_out/s6
timeout 2400 python -m pytest tests -m gpu -q -rs --timeout 1500 > gpurun_out/s6/gpu_tests.log 2>&1; tail -4 gpurun_out/s6/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6/smoke.log 2>&1; tail -2 gpurun_out/s6/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --stages > gpurun_out/s6/bench_cluster2B.json 2> gpurun_out/s6/bench.err; tail -c 600 gpurun_out/s6/bench_cluster2B.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s6/bench_reference.json 2>> gpurun_out/s6/bench.err; tail -c 300 gpurun_out/s6/bench_reference.json
