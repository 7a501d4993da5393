timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
bash scripts/gpu_cluster.sh
timeout 900 python bench.py --config scene500M --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_scene.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_scene.json'));print('scene500M',round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
