timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_color_filter.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_color_filter.json'));print('terrain',round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
timeout 900 python bench.py --config cluster2B --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cluster.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_cluster.json'));print('cluster2B',round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
