set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_large.py -m gpu -q -x -rs --timeout 1200 -k "many_leaves or two_pass or cluster or stadium or scene" > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
CONFIGS="cluster2B" bash scripts/gpu_launches.sh
