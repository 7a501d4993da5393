set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KERNELS="k_count|k_dist_hist" COUNT=3 TAG=split_r02 CONFIG=cluster2B bash scripts/gpu_ncu.sh
KERNELS="k_scatter|k_occupy|k_prefix|k_finalize" COUNT=20 TAG=voxelize_r02 CONFIG=terrain20M bash scripts/gpu_ncu.sh
