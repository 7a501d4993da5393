timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2>gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launches3.py gpurun_out/launches.csv > gpurun_out/launches3.txt; head -12 gpurun_out/launches3.txt
