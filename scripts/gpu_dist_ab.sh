# distribute rewrite: parity, then A/B of the scatter variants, then a launch list
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for v in 0 1 2; do
  LOD_DIST_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_v$v.json'));print('var $v', round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
done
LOD_DIST_VARIANT=${BEST:-0} timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "k_dist|k_count|k_bounds" gpurun_out/launches.csv | tail -12 | cut -c1-40,120-400
