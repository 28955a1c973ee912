# same-box A/B of an environment switch: bench.py with and without $AB_ENV, alternating
mkdir -p gpurun_out
show() {
  python -c "
import json,sys
j=json.loads(sys.stdin.read()); k=j['kernels']; s=j['steps']
print('$1', round(j['ms_per_step'],3), round(j['e2e']['ms_per_step'],3), ' '.join(f'{n}={v[\"ms_total\"]/s:.3f}' for n,v in list(k.items())[:${AB_TOPK:-5}]))"
}
for wl in ${AB_WORKLOADS:-pr tc}; do
  for r in 1 2; do
    timeout 600 python bench.py --no-cpu-baseline --no-extras --workload $wl --steps ${AB_STEPS:-20} 2>/dev/null | show "$wl base"
    env $AB_ENV timeout 600 python bench.py --no-cpu-baseline --no-extras --workload $wl --steps ${AB_STEPS:-20} 2>/dev/null | show "$wl $AB_ENV"
  done
done
