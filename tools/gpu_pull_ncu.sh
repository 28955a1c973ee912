# ncu --set full of one real (non-no-op) k_pr_pull_fused launch of a C2 batch
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-extras --workload pr"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pr_pull_fused --csv \
  --log-file gpurun_out/pull_list.csv $CMD > /dev/null 2>&1
idx=$(python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/pull_list.csv")))
h=next(i for i,r in enumerate(rows) if "Kernel Name" in r)
v=[float(r[rows[h].index("Metric Value")].replace(",","")) for r in rows[h+1:]]
unit=rows[h+1][rows[h].index("Metric Unit")]
big=[i for i,x in enumerate(v) if x > (100000 if unit=="ns" else 100)]
print(big[-2] if len(big)>1 else (big[-1] if big else 0))
PY
)
echo "pull launch index $idx"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pr_pull_fused -s $idx -c 1 \
   -o gpurun_out/prof_pull_pr $CMD > gpurun_out/ncu_pull.log 2>&1
echo "ncu rc=$?"
