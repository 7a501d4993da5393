# compute-sanitizer over the round-2 stage-level API and pipelining paths (extract.cu kernels,
# lod_merge_pyramid, the staged Partitioner through lod_dist_*, lod_tree_set_output_wait,
# in-place receive) -> gpurun_out/sanitize_stage_*.log
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SEL='(merge or count or stadium_30000 or blobs_150000_11 or extract_equals_oracle and 1000 or projection or sample_node or one_tree or distributed_matches) and not multiprocess'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_stages.py tests/test_gpu_sampling_stages.py tests/test_gpu_pipeline.py tests/test_dist_gpu.py \
    -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_stage_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_stage_summary.txt
  tail -3 gpurun_out/sanitize_stage_$tool.log >> gpurun_out/sanitize_stage_summary.txt
done
cat gpurun_out/sanitize_stage_summary.txt
