mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_dist_local_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
AB_TOPK=2 AB_WORKLOADS="pr tc" AB_ENV=GD_UPLOAD_EARLY=1 bash tools/gpu_ab_env.sh
