# ncu --set full of the distribute kernels (one build, terrain20M)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dist_rank|k_dist_scatter" -s 2 -c 2 -o gpurun_out/prof_rank -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_rank.log 2>&1
tail -3 gpurun_out/ncu_rank.log
