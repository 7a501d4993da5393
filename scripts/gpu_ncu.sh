# ncu --set full of selected kernels of one build -> gpurun_out/<tag>.ncu-rep (+ text summary)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KERNELS}" -c ${COUNT:-4} \
  -o gpurun_out/${TAG:-prof} python scripts/one_build.py --config ${CONFIG:-cluster2B} --builds 1 > gpurun_out/${TAG:-prof}.log 2>&1
tail -3 gpurun_out/${TAG:-prof}.log
python scripts/ncu_summary.py gpurun_out/${TAG:-prof}.ncu-rep > gpurun_out/${TAG:-prof}_summary.txt 2>&1; head -80 gpurun_out/${TAG:-prof}_summary.txt
