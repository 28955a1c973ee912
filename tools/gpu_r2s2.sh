mkdir -p gpurun_out
BENCH_ARGS="--no-extras --steps 20" bash tools/gpu_variants.sh
