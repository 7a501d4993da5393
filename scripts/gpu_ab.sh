# A/B of voxelizer library variants (scripts/build_variant.py) -> gpurun_out/s6/ab_<tag>.txt
mkdir -p gpurun_out/s6
CONFIGS="${CONFIGS:-cluster2B terrain20M scene500M}" LIBS="$LIBS" bash scripts/ab_lib.sh 2>&1 | tee gpurun_out/s6/ab_$TAG.txt
