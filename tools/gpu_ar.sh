#!/bin/bash
# NVLink all-reduce micro-benchmarks on a multi-GPU box: n_tok sweep of the push kernel, NCCL and torch symm-mem.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -gt $N ] && continue
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) \
    tools/ar_bench.py --sweep > gpurun_out/ar_tp$n.log 2>&1; echo "tp=$n rc=$?"; grep -E "us/call|multicast|unavailable|symm_mem" gpurun_out/ar_tp$n.log | sort -u
done
