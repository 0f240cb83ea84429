#!/bin/bash
# Interleaved A/B of two engine settings on one TP stage (tools/ab_dist.py) at TP=4 and TP=2, 70B layers.
# usage: gpurun --gpus 4 -- 'A=HX_X=0 B=HX_X=1 bash tools/gpu_ab_dist.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 600 python -m pytest $TESTS -q -rf > gpurun_out/abd_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/abd_tests.log; fi
for tp in ${TPS:-4 2}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $tp --master-addr 127.0.0.1 \
    --master-port $((29700 + tp)) tools/ab_dist.py --tp $tp --layers 40 --a "$A" --b "$B" > gpurun_out/abd_tp$tp.log 2>&1
  echo "tp=$tp rc=$?"; grep -E "p50" gpurun_out/abd_tp$tp.log
done
