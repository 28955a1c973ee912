mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not test_c2_pagerank_all and not c3_tc and not c4_grid" 2>&1 | tail -2
AB_TOPK=2 AB_WORKLOADS="pr tc" AB_STEPS=10 AB_ENV=GD_ALLOC_EXACT=1 bash tools/gpu_ab_env.sh
for e in "" "GD_ALLOC_EXACT=1"; do
  env $e timeout 900 python bench.py --no-cpu-baseline --no-extras --workload tc-rmat24 --percent 5 --steps 5 --warmup 3 --e2e-steps 3 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); s=j['steps']
print('tc-rmat24 5% $e', round(j['ms_per_step'],2), 'e2e', round(j['e2e']['ms_per_step'],2), 'kernels', round(sum(v['ms_total'] for v in j['kernels'].values())/s,2))"
done
