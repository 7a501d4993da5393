# full evidence run on one B200 -> gpurun_out/ (copied to profiles/<tag>/ afterwards)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_terrain20M_color_filter.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
for m in random first-come weighted; do
  timeout 600 python bench.py --steps 10 --warmup 3 --mode $m --no-cpu-baseline --no-e2e > gpurun_out/bench_terrain20M_$m.json 2>> gpurun_out/bench.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --config scene500M --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_scene500M_color_filter.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --config scene500M --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --points 1000000000 > gpurun_out/bench_scene1B_color_filter.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --config cluster2B --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cluster2B_color_filter.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launches3.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_dist_scatter|k_dist_hist|k_scatter|k_finalize|k_occupy|k_prefix|k_count" -s 72 -c 12 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
