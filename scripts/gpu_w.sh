timeout 900 python -m pytest tests -m gpu -x -q -k "weighted or edge" > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --mode weighted > gpurun_out/bench_w.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_w.json'));print('weighted',round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
