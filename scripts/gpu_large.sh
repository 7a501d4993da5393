# large-config benches (device-resident value only), one at a time, bounded
run() { echo "== $*"; timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/large.json 2> gpurun_out/large.err; tail -c 600 gpurun_out/large.err; python -c "
import json;d=json.load(open('gpurun_out/large.json'));print(round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],2),'ms', {k:round(x,2) for k,x in d['stages_ms'].items()}, d['tree'])" 2>/dev/null; nvidia-smi --query-gpu=memory.used --format=csv,noheader; }
run --config scene500M --steps 3 --warmup 3
run --config scene500M --steps 3 --warmup 3 --points 1000000000
run --config scene500M --steps 3 --warmup 3 --mode random
run --config cluster2B --steps 3 --warmup 3
