# compute-sanitizer over a subset of the -m gpu parity tests: the store
# (delete/add/merge kernels), SSSP (cooperative fixpoints with grid barriers
# and warp-aggregated queue appends), PR (fused pull, device loop state), TC
# (shared-memory merge, hub bitmaps) and the flood.  One GPU.
mkdir -p gpurun_out
SEL="figure or parallel or rw3 or rw150 or rwL1000 or sssp_worked or sssp_r1 or sssp_r2 or sssp_und_repro or sssp_und3 or sssp_multi1 or pr_r1 or pr_r2 or tc_r1 or tc_r2 or tc_multi3 or tc_omp0 or propagate_flags or hub_bitmaps or (near_far and grid and 100)"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 2400 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider -k "$SEL" \
     > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3
done
