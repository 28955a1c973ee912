mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_local_gpu.py -x -q -p no:cacheprovider -k "flood or pr or propagate" 2>&1 | tail -2
AB_TOPK=9 AB_WORKLOADS="pr" AB_ENV=GD_FLOOD_COMPRESS=1 bash tools/gpu_ab_env.sh
