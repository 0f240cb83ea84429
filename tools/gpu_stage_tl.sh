#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/stl
for tp in ${TPS:-4 2}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $tp --master-addr 127.0.0.1 \
    --master-port $((29600 + tp)) tools/stage_timeline.py --tp $tp --layers 20 > gpurun_out/stl/tp$tp.txt 2>&1
  echo "tp=$tp rc=$?"; grep -v Warn gpurun_out/stl/tp$tp.txt | tail -8
done
