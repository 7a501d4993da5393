timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not large" > gpurun_out/par.log 2>&1; tail -2 gpurun_out/par.log
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/dist.log 2>&1; tail -30 gpurun_out/dist.log
