# A/B: bench the working tree and a stash of the previous build, 3 runs each
set -x
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('B', j['ms_per_step'], j['e2e']['ms_per_step'])"
  if [ -d /tmp/prev ]; then true; fi
  if [ -f prev/libgdb200.so ]; then cp paper_2507_11094_b200/libgdb200.so /tmp/cur.so; cp prev/libgdb200.so paper_2507_11094_b200/libgdb200.so;
    timeout 600 python bench.py --no-cpu-baseline --steps 20 ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('A', j['ms_per_step'], j['e2e']['ms_per_step'])";
    cp /tmp/cur.so paper_2507_11094_b200/libgdb200.so; fi
done
