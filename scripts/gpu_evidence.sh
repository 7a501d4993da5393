# round evidence on one B200 -> gpurun_out/ (copied to profiles/r02/ afterwards)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
timeout 2400 python -m pytest tests -m gpu -q -rs --timeout 1500 > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --stages > gpurun_out/bench_cluster2B_color_filter.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --config scene500M --points 1000000000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_scene1B_color_filter.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --config scene500M --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --mode random > gpurun_out/bench_scene500M_random.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --config scene500M --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_scene500M_color_filter.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --config terrain20M --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_terrain20M_color_filter.json 2>> gpurun_out/bench.err
for m in random first-come weighted; do
  timeout 600 python bench.py --config terrain20M --steps 10 --warmup 3 --mode $m --no-cpu-baseline --no-e2e > gpurun_out/bench_terrain20M_$m.json 2>> gpurun_out/bench.err
done
CONFIGS="cluster2B terrain20M" bash scripts/gpu_launches.sh
[ -n "$SANITIZE" ] && bash scripts/sanitize.sh
true
