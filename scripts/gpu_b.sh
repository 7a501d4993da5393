# bench + launch list only (no tests)
m=${1:-color_filter}
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --mode $m > gpurun_out/bench_$m.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_$m.json'));print('$m',round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --mode $m > /dev/null 2>&1
python scripts/launches3.py gpurun_out/launches_q.csv > gpurun_out/launches_q.txt; head -12 gpurun_out/launches_q.txt
