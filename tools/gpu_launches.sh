# plain run, then the same command under ncu for the per-launch device times
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 2 --no-cpu-baseline ${BENCH_ARGS}"
timeout 600 $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/plain.err; cat gpurun_out/plain.json | head -c 600; echo; tail -3 gpurun_out/ncu.log
