# tests + smoke, bench, then the launch list of a short bench under ncu
bash tools/gpu_check.sh
BENCH_ARGS="--no-cpu-baseline ${BENCH_ARGS}" bash tools/gpu_bench.sh
if [ -n "$LAUNCHES" ]; then bash tools/gpu_launches.sh; fi
