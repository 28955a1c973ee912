timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload sssp --steps 10 --warmup 3 --static > gpurun_out/b_sssp_static.json 2> gpurun_out/b_sssp_static.err; echo "rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/b_sssp_static.json')); print(j['ms_per_step'], j.get('static'))"
