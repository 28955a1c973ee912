mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not test_c2_pagerank_all and not c3_tc and not c4_grid" 2>&1 | tail -2
AB_TOPK=2 AB_WORKLOADS="pr tc" AB_STEPS=10 AB_ENV=GD_INDEX_FULL_SORT=1 bash tools/gpu_ab_env.sh
