# the N>1 code path at world size 1 (torchrun, NCCL, partitioned PR / SSSP
# stores, replicated TC with record slices), one GPU
mkdir -p gpurun_out
for wl in pr sssp tc sssp-grid; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --force-dist --workload $wl --no-extras --no-cpu-baseline --steps 5 --warmup 3 \
    > gpurun_out/forcedist_$wl.json 2> gpurun_out/forcedist_$wl.err
  echo "$wl rc=$?"
  python -c "
import json; j=json.loads([l for l in open('gpurun_out/forcedist_$wl.json') if l.startswith('{')][-1]); print('$wl', round(j['ms_per_step'],3), 'ms', j['config']['parallelism'][:60], j.get('comm'))" 2>&1 | tail -1
done
