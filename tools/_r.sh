timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "tc or TC or smoke or golden or comm" 2>&1 | tail -1
for p in 1 10; do timeout 900 python bench.py --workload tc-rmat24 --percent $p --steps 3 --warmup 2 --e2e-steps 2 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err; python -c "
import json; j=json.load(open('gpurun_out/t.json')); print('tc24 $p%', j['ms_per_step'], {k: round(v['ms_total']/j['steps'],2) for k,v in j['kernels'].items()})"; done
timeout 900 python bench.py --workload tc --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err; python -c "
import json; j=json.load(open('gpurun_out/t.json')); print('C3', j['ms_per_step'], {k: round(v['ms_total']/j['steps'],2) for k,v in j['kernels'].items()})"
