#!/bin/bash
# Multi-GPU bench lines (70B asymmetric plans) on a gpurun --gpus 4 box.
# usage: gpurun --gpus 4 --timeout 1800 -- bash tools/gpu_multi.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 2 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  echo "N=$N rc=$?"; tail -1 gpurun_out/bench_n$N.json | cut -c1-400
done
