mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_dist_local_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for wl in pr pr tc sssp-grid; do
timeout 600 python bench.py --no-cpu-baseline --no-extras --workload $wl --steps 10 2>/dev/null | python -c "
import json,sys
j=json.loads(sys.stdin.read())
print('$wl', round(j['ms_per_step'],3), 'e2e', round(j['e2e']['ms_per_step'],3), j['e2e']['h2d_bytes_per_step'], j['e2e']['api'])"
done
