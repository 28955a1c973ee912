# plain run, then one ncu --set full capture of the named kernels (1 GPU)
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline ${BENCH_ARGS}"
timeout 600 $CMD > gpurun_out/plain_full.json 2> gpurun_out/plain_full.err && \
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-6} \
   -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
tail -5 gpurun_out/ncu_full.log
