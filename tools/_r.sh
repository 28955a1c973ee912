timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "sssp or SSSP or smoke or golden or c1" 2>&1 | tail -1
for p in 1 10; do timeout 900 python bench.py --workload sssp-rmat24 --percent $p --steps 4 --warmup 2 --e2e-steps 2 --no-cpu-baseline > gpurun_out/s.json 2> gpurun_out/s.err; python -c "
import json; j=json.load(open('gpurun_out/s.json')); print('p=$p', round(j['ms_per_step'],2), {k: round(v['ms_total']/j['steps'],2) for k,v in j['kernels'].items()})"; done
timeout 900 python bench.py --workload sssp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s.json 2> gpurun_out/s.err; python -c "
import json; j=json.load(open('gpurun_out/s.json')); print('C1', round(j['ms_per_step'],3), {k: round(v['ms_total']/j['steps'],3) for k,v in j['kernels'].items()})"
