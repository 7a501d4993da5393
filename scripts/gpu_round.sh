# full round check on one B200: gpu tests, smoke, bench lines, launch list, ncu --set full of the top kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --steps 10 --warmup 3 --mode random --no-cpu-baseline > gpurun_out/bench_random.json 2> gpurun_out/bench_random.err; cat gpurun_out/bench_random.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1; tail -3 gpurun_out/launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_radix|k_count|k_occupy|k_scatter|k_finalize|k_bounds" -s 40 -c 8 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
