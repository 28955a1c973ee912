# north_star target sweep: R-MAT scale-24, PR / SSSP / TC at 1/5/10/20% batches (1 GPU)
mkdir -p gpurun_out/sweep
for wl in pr-rmat24 sssp-rmat24 tc-rmat24; do
  for p in 1 5 10 20; do
    timeout 900 python bench.py --workload $wl --percent $p --steps 5 --warmup 3 --e2e-steps 3 --no-cpu-baseline \
      > gpurun_out/sweep/${wl}_p${p}.json 2> gpurun_out/sweep/${wl}_p${p}.err
    echo "$wl $p rc=$?"
  done
done
