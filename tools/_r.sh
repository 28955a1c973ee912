timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q --timeout 300 -p no:cacheprovider -k "pr or PR or c2 or comm" > gpurun_out/pytest_pr.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pr.log
bash tools/gpu_ab.sh 2>&1 | grep "^[AB] "
