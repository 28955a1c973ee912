mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "pr and not test_c2_pagerank_all" 2>&1 | tail -2
BENCH_ARGS="--no-extras --steps 20" bash tools/gpu_variants.sh
