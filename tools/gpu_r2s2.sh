mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_dist_local_gpu.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
AB_TOPK=2 AB_WORKLOADS="pr tc sssp-grid" AB_STEPS=8 AB_ENV=GD_UPLOAD_EARLY=1 bash tools/gpu_ab_env.sh
