for dm in 0 1; do for p in 1 10 20; do GD_SSSP_DECR=$dm timeout 900 python bench.py --workload sssp-rmat24 --percent $p --steps 4 --warmup 2 --e2e-steps 2 --no-cpu-baseline > gpurun_out/s.json 2> gpurun_out/s.err; python -c "
import json; j=json.load(open('gpurun_out/s.json')); print('decr=$dm p=$p', round(j['ms_per_step'],2), {k: round(v['ms_total']/j['steps'],2) for k,v in j['kernels'].items()})"; done
GD_SSSP_DECR=$dm timeout 900 python bench.py --workload sssp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s.json 2> gpurun_out/s.err; python -c "
import json; j=json.load(open('gpurun_out/s.json')); print('decr=$dm C1', round(j['ms_per_step'],3))"; done
