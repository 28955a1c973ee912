bash tools/gpu_launches.sh > gpurun_out/launches.log 2>&1; echo "launches rc=$?"; tail -2 gpurun_out/launches.log
KREGEX='k_pr_pull_fused|k_edit_base|k_del_scan|k_pr_contrib|k_aff_sample' NCU_SKIP=4 NCU_COUNT=12 bash tools/gpu_ncu_full.sh > gpurun_out/full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/full.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; cat gpurun_out/bench_default.json | head -c 300
