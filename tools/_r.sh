mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_parity.log
bash tools/gpu_ab.sh 2>&1 | grep "^[AB] "
