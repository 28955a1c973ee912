timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
bash tools/gpu_launches.sh > gpurun_out/launches.log 2>&1; echo "launches rc=$?"
KREGEX='k_pr_pull_fused|k_edit_base|k_del_scan|k_pr_contrib|k_aff_sample' NCU_SKIP=4 NCU_COUNT=12 bash tools/gpu_ncu_full.sh > gpurun_out/full.log 2>&1; echo "full rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
for w in sssp tc sssp-grid; do timeout 1200 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"; done
