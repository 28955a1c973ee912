mkdir -p gpurun_out
start=$(date +%s)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not test_c2_pagerank_all" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - start ))s"
tail -3 gpurun_out/pytest_gpu.log
GD_SSSP_DEBUG=1 timeout 600 python tools/sssp_diag.py grid 4 2>&1 | grep -v Warn | tail -9
for wl in sssp-grid sssp; do
timeout 600 python bench.py --no-cpu-baseline --no-extras --workload $wl --steps 6 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read()); k=j['kernels']; s=j['steps']
print('$wl', round(j['ms_per_step'],3), round(j['e2e']['ms_per_step'],3), j['roofline']['frac'], ' '.join(f'{n}={v[\"ms_total\"]/s:.3f}' for n,v in list(k.items())[:5]))"
done
