# ncu launch lists (time + DRAM bytes per kernel) of the last build -> gpurun_out/launches_<config>.{csv,txt}
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${CONFIGS:-cluster2B}; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$c.csv python scripts/one_build.py --config $c --builds 2 > gpurun_out/launches_$c.log 2>&1
  python scripts/launches3.py gpurun_out/launches_$c.csv > gpurun_out/launches_$c.txt 2>&1; head -40 gpurun_out/launches_$c.txt
done
