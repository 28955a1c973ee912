free -g | head -2
timeout 1500 python bench.py --workload pr-c5 --steps 3 --warmup 2 --e2e-steps 2 --no-cpu-baseline > gpurun_out/c5pr.json 2> gpurun_out/c5pr.err; echo "pr-c5 rc=$?"; tail -4 gpurun_out/c5pr.err
python -c "
import json; j=json.load(open('gpurun_out/c5pr.json')); print(j['ms_per_step'], j['value'], j['e2e']['ms_per_step'], j['roofline']['kernel'], j['roofline']['frac'], {k: round(v['ms_total']/j['steps'],2) for k,v in j['kernels'].items()})"
timeout 1500 python bench.py --workload sssp-c5 --steps 3 --warmup 2 --e2e-steps 2 --no-cpu-baseline > gpurun_out/c5sssp.json 2> gpurun_out/c5sssp.err; echo "sssp-c5 rc=$?"; tail -4 gpurun_out/c5sssp.err
python -c "
import json; j=json.load(open('gpurun_out/c5sssp.json')); print(j['ms_per_step'], j['value'], j['e2e']['ms_per_step'], j['roofline']['kernel'], {k: round(v['ms_total']/j['steps'],2) for k,v in j['kernels'].items()})"
