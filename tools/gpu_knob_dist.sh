#!/bin/bash
# One process per setting of a C-side knob (read once at library load), TP stage A/B on one box:
# usage: gpurun --gpus 4 -- 'KNOB=HX_AR_BATCHPOLL VALUES="1 0 1 0" TPS="4" bash tools/gpu_knob_dist.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tp in ${TPS:-4}; do for v in $VALUES; do
  env $KNOB=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $tp --master-addr 127.0.0.1 \
    --master-port $((29800 + tp)) tools/ab_dist.py --tp $tp --layers 40 --rounds 3 > gpurun_out/knob_tp${tp}_$v.log 2>&1
  echo "tp=$tp $KNOB=$v: $(grep -E '^A ' gpurun_out/knob_tp${tp}_$v.log | sed 's/.*p50 decode step //')"
done; done
