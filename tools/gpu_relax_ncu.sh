# ncu --set full of one batch-phase k_fixpoint<0> (RELAX) launch of the C4 grid bench
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-extras --workload sssp-grid"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fixpoint --csv \
  --log-file gpurun_out/fp_list.csv $CMD > /dev/null 2>&1
idx=$(python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/fp_list.csv")))
h=next(i for i,r in enumerate(rows) if "Kernel Name" in r)
hd=rows[h]
L=[(r[hd.index("Kernel Name")], float(r[hd.index("Metric Value")].replace(",",""))) for r in rows[h+1:]]
print(sum(1 for k,_ in L), file=open("gpurun_out/fp_count.txt","w"))
for i,(k,v) in enumerate(L): print(i, k[:40], v, file=open("gpurun_out/fp_idx.txt","a"))
relax=[i for i,(k,v) in enumerate(L) if "k_fixpoint<0>" in k or "k_fixpoint<(int)0>" in k]
print(relax[-2] if len(relax)>1 else 0)
PY
)
echo "relax launch index $idx"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fixpoint -s $idx -c 1 \
   -o gpurun_out/prof_relax_grid $CMD > gpurun_out/ncu_relax.log 2>&1
echo "ncu rc=$?"
