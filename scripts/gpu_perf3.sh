# parity + terrain bench + scene/cluster benches
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
run() { echo "== $*"; timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/large.json 2> gpurun_out/large.err; tail -c 300 gpurun_out/large.err; python -c "
import json;d=json.load(open('gpurun_out/large.json'));print(round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],2),'ms', {k:round(x,2) for k,x in d['stages_ms'].items()})" 2>/dev/null; }
run --steps 10 --warmup 3
run --config scene500M --steps 3 --warmup 3 --points 1000000000
run --config cluster2B --steps 3 --warmup 3
