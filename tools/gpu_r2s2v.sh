# A/B of the merge-copy variants on C2 and C3
mkdir -p gpurun_out
BENCH_ARGS="--no-extras" bash tools/gpu_variants.sh
BENCH_ARGS="--no-extras --workload tc --steps 6" bash tools/gpu_variants.sh
