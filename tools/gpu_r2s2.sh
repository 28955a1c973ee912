mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "sssp and not test_c2_pagerank_all" 2>&1 | tail -2
AB_TOPK=6 AB_WORKLOADS="sssp-grid" AB_STEPS=6 AB_ENV=GD_SSSP_G=8 bash tools/gpu_ab_env.sh
