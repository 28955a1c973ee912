timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu_ab.sh 2>&1 | grep "^[AB] "
timeout 600 python tools/timeline.py pr 4 > gpurun_out/timeline_pr.log 2>&1; rm -f gpurun_out/trace.json
grep "batch\|span" gpurun_out/timeline_pr.log | head -6
