mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not test_c2_pagerank_all and not c3_tc and not c4_grid" 2>&1 | tail -2
BENCH_ARGS="--no-extras --steps 20" bash tools/gpu_variants.sh
BENCH_ARGS="--no-extras --workload tc --steps 6" bash tools/gpu_variants.sh
