mkdir -p gpurun_out
start=$(date +%s)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not test_c2_pagerank_all" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - start ))s"
tail -3 gpurun_out/pytest_gpu.log
AB_TOPK=3 AB_WORKLOADS="pr tc" AB_ENV=GD_READ_SYNC=1 bash tools/gpu_ab_env.sh
