# A/B: bench the working tree (B) and prev/libgdb200.so (A), 3 runs each;
# prints step ms, e2e ms and the per-batch ms of the main kernels
set -x
mkdir -p gpurun_out
show() {
  python -c "
import json,sys
j=json.loads(sys.stdin.read()); k=j['kernels']; s=j['steps']
print('$1', round(j['ms_per_step'],3), round(j['e2e']['ms_per_step'],3), ' '.join(f'{n}={v[\"ms_total\"]/s:.3f}' for n,v in list(k.items())[:6]))"
}
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} 2>/dev/null | show B
  if [ -f prev/libgdb200.so ]; then cp paper_2507_11094_b200/libgdb200.so /tmp/cur.so; cp prev/libgdb200.so paper_2507_11094_b200/libgdb200.so;
    timeout 600 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} 2>/dev/null | show A
    cp /tmp/cur.so paper_2507_11094_b200/libgdb200.so; fi
done
