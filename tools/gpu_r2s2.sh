# round-2 session-2: GPU tests (without the 8-minute C2 reference runs), e2e probe, C2 + C3 benches
mkdir -p gpurun_out
start=$(date +%s)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not test_c2_pagerank_all" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - start ))s"
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python tools/e2e_probe2.py 2>&1 | grep -v Warn | tail -12
for wl in pr tc; do
timeout 600 python bench.py --no-cpu-baseline --no-extras --workload $wl > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; echo "bench $wl rc=$?"
python - <<PY
import json; d=json.load(open("gpurun_out/bench_$wl.json"))
print("$wl", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3), {k:(round(v["ms_total"]/v["launches"],4), v["gbs"] and round(v["gbs"])) for k,v in d["kernels"].items()})
PY
done
