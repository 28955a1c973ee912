timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "tc or TC or smoke or golden" 2>&1 | tail -1
for wl in tc-rmat24 tc; do timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/tcx.json 2> gpurun_out/tcx.err; python -c "
import json; j=json.load(open('gpurun_out/tcx.json')); print('$wl', j['ms_per_step'], j['e2e']['ms_per_step'], j['roofline']['kernel'], j['roofline']['frac'], {k: (round(v['ms_total']/j['steps'],2), v['gbs']) for k,v in j['kernels'].items()})"; done
