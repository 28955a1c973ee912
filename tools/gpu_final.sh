# the driver's round-end steps: full -m gpu suite (timed), smoke, the default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
start=$(date +%s)
timeout 1150 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=12 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - start ))s"
tail -20 gpurun_out/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
grep "e2e\|reference\]" gpurun_out/bench.err | tail -8
python - <<'PY'
import json; d=json.load(open("gpurun_out/bench.json"))
print("C2", round(d["ms_per_step"],3), "e2e", round(d["e2e"]["ms_per_step"],3), "frac", round(d["roofline"]["frac"],3), "cpu", d["cpu_baseline"]["value"])
for k,v in d["extras"].items(): print(k, round(v["ms_per_step"],3), "e2e", round(v["e2e"]["ms_per_step"],3), v["roofline"]["kernel"], round(v["roofline"]["frac"],3))
PY
