mkdir -p gpurun_out/c5
for wl in pr-c5 sssp-c5; do
  timeout 1200 python bench.py --workload $wl --no-extras --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/c5/$wl.json 2> gpurun_out/c5/$wl.err
  echo "$wl rc=$?"
  python -c "
import json; j=json.loads(open('gpurun_out/c5/$wl.json').read().strip().splitlines()[-1]); s=j['steps']
print('$wl', round(j['ms_per_step'],2), 'e2e', round(j['e2e']['ms_per_step'],2), {k: round(v['ms_total']/s,2) for k,v in list(j['kernels'].items())[:5]})"
done
