# launch list of one scene500M build (2-pass distribute, extensions, deep trees)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_scene.csv python bench.py --config scene500M --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scene_ncu.log 2>&1
python scripts/launches3.py gpurun_out/launches_scene.csv > gpurun_out/launches_scene.txt; head -30 gpurun_out/launches_scene.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
