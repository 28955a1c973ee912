timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_par.log
bash tools/gpu_ab.sh 2>&1 | grep "^[AB] "
