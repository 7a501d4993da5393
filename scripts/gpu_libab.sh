# A/B of prebuilt library variants in scratch/*.so: bench + per-kernel DRAM bytes
for f in scratch/*.so; do
  cp $f paper_2302_14801_b200/_lib/liblodb200.so
  echo "== $f"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print(round(d['value']/1e9,3),'G/s', {k:round(x,3) for k,x in d['stages_ms'].items()})"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/l.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python scripts/launches3.py gpurun_out/l.csv | head -8
done
