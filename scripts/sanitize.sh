# compute-sanitizer passes over the quick golden cases (<= 300k points) -> gpurun_out/sanitize_*.log
# memcheck: out-of-bounds / misaligned global+shared accesses, leaks of device allocations;
# racecheck: shared-memory hazards; synccheck: illegal barrier use.  Every kernel of the
# library (split, distribute incl. the 2-pass and leaf-id paths, voxelize in all four
# strategies, encode, ingest, checks) runs under each tool.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SEL='(part_ or small_tree or identical or maxface or sparse or single_point or initial6 or depth_limit or uniform_300k or many_leaves_400k or cluster1500k or test_device_pack or test_nccl) and not multiprocess'
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_errors.py tests/test_gpu_upload.py tests/test_dist_gpu.py \
    -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
