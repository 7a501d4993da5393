set -x
timeout 300 python -m pytest tests/test_gpu_generators.py -q > gpurun_out/gen.log 2>&1; tail -3 gpurun_out/gen.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 600 python bench.py --steps 5 --warmup 3 --mode random --no-cpu-baseline > gpurun_out/bench1r.json 2> gpurun_out/bench1r.err; cat gpurun_out/bench1r.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_voxelize|k_radix|k_count" -s 30 -c 6 -o gpurun_out/prof1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log
