mkdir -p gpurun_out
bash tools/gpu_forcedist.sh
# the driver's multi-GPU launch at N=1 without --force-dist, and the reference arm
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 3 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/tr1.json 2> gpurun_out/tr1.err; echo "torchrun N=1 rc=$?"; tail -c 300 gpurun_out/tr1.json
