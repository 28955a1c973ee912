# Bench the working-tree library and each variants/libgdb200_*.so (same
# sources, different compile-time knobs); prints step ms, e2e ms, top kernels.
mkdir -p gpurun_out
show() {
  python -c "
import json,sys
j=json.loads(sys.stdin.read()); k=j['kernels']; s=j['steps']
print('$1', round(j['ms_per_step'],3), round(j['e2e']['ms_per_step'],3), ' '.join(f'{n}={v[\"ms_total\"]/s:.3f}' for n,v in list(k.items())[:4]))"
}
cp paper_2507_11094_b200/libgdb200.so /tmp/base.so
for r in 1 2; do
  for v in /tmp/base.so variants/libgdb200_*.so; do
    cp $v paper_2507_11094_b200/libgdb200.so
    timeout 600 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} 2>/dev/null | show $(basename $v)
  done
done
cp /tmp/base.so paper_2507_11094_b200/libgdb200.so
