# near-far bucket width A/B on the grid (configs[3]): GD_SSSP_DELTA overrides
# the 3x-mean-weight default
for r in 1; do
for dl in default 40 75 150 300 600; do
  if [ $dl = default ]; then unset GD_SSSP_DELTA; else export GD_SSSP_DELTA=$dl; fi
  timeout 600 python bench.py --workload sssp-grid --no-extras --no-cpu-baseline --steps 4 --warmup 3 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); k=j['kernels']; s=j['steps']
print('delta=$dl', round(j['ms_per_step'],2), ' '.join(f'{n}={v[\"ms_total\"]/s:.2f}' for n,v in list(k.items())[:5]))"
done; done
