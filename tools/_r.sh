bash tools/gpu_ab.sh 2>&1 | grep "^[AB] "
timeout 900 python bench.py --workload tc --steps 3 --warmup 3 > gpurun_out/tcref.json 2> gpurun_out/tcref.err; echo "tc rc=$?"; grep reference gpurun_out/tcref.err; python -c "
import json; j=json.load(open('gpurun_out/tcref.json')); print(j['ms_per_step'], j['cpu_baseline'])"
