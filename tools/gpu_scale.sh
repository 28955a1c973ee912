set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale.py -m gpu -q -x --timeout 900 -p no:cacheprovider -s > gpurun_out/pytest_scale.log 2>&1; echo "scale rc=$?"
tail -15 gpurun_out/pytest_scale.log
for wl in sssp tc sssp-grid; do
  timeout 900 python bench.py --no-cpu-baseline --workload $wl --steps 3 --warmup 1 --e2e-steps 1 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; echo "$wl rc=$?"
  tail -2 gpurun_out/bench_$wl.err; head -c 400 gpurun_out/bench_$wl.json; echo
done
