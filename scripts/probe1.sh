mkdir -p gpurun_out
(free -g; nproc; nvidia-smi; df -h /tmp /dev/shm; ulimit -l) > gpurun_out/box.txt 2>&1
timeout 600 python bench.py --config cluster2B --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --stages > gpurun_out/p1_cluster2B.json 2> gpurun_out/p1.err
timeout 600 python bench.py --config scene500M --points 1000000000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --stages > gpurun_out/p1_scene1B.json 2>> gpurun_out/p1.err
