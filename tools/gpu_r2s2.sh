mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tc and not test_c2_pagerank_all" 2>&1 | tail -2
AB_TOPK=3 AB_WORKLOADS="tc" AB_STEPS=6 AB_ENV=GD_TC_META=0 bash tools/gpu_ab_env.sh
