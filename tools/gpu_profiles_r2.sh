# Round-2 profile set (one GPU), one piece per call (gpurun returns at most
# 64 MiB): PROFILE=launches -> the launch list of the C2 default bench;
# PROFILE=<workload> -> one `ncu --set full` capture of its top kernels,
# after the same command ran clean without ncu.
set -x
mkdir -p gpurun_out
if [ "$PROFILE" = launches ]; then
  BENCH_ARGS="--no-extras" bash tools/gpu_launches.sh
  rm -f gpurun_out/plain.err
  exit 0
fi
case $PROFILE in
  pr) kre="k_edit_base|k_pr_pull_fused|k_del_scan|k_aff_sample"; cnt=8;;
  tc) kre="k_tc_merge|k_edit_base"; cnt=4;;
  sssp-grid) kre="k_fixpoint"; cnt=4;;
esac
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-extras --workload $PROFILE"
timeout 900 $CMD > /tmp/plain.json 2> /tmp/plain.err && \
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 6 -c $cnt \
   -o gpurun_out/prof_$PROFILE $CMD > gpurun_out/ncu_$PROFILE.log 2>&1
echo "$PROFILE rc=$?"
ls -la gpurun_out
