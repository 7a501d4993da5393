# racecheck / memcheck of the round-2 shared-memory kernels: TMA scatter (2-pass distribute),
# hot-counter caches (count, extension rounds), extension list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in racecheck memcheck; do
timeout 2400 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "many_leaves_400k or cluster1500k or initial6_ext3 or identical_2000" -p no:cacheprovider \
  > gpurun_out/sanitize_${tool}_r02kernels.log 2>&1
echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_${tool}_r02kernels.log
done
