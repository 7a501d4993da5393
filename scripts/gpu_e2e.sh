timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err
python -c "import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(round(d['value']/1e9,3),'G/s e2e',round(d['e2e']['value']/1e9,3), d['e2e']['ms_per_step'])"
