timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1; tail -3 gpurun_out/par.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
SKIP=0 COUNT=1 bash scripts/gpu_prof.sh k_scatter
SKIP=0 COUNT=1 bash scripts/gpu_prof.sh k_occupy
SKIP=1 COUNT=1 bash scripts/gpu_prof.sh k_finalize
