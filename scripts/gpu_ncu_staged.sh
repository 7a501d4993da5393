timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dist_scatter_staged" -s 1 -c 1 -o gpurun_out/prof_staged -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_staged.log 2>&1
tail -2 gpurun_out/ncu_staged.log
