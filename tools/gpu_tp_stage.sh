#!/bin/bash
# TP=4 / TP=2 x 40-layer 70B stage times (tools/ab_dist.py, deferred QKV off vs on) + TP=4 attention timeline
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tps
python tools/attn_timeline.py llama2-70b --tp=4 > gpurun_out/tps/tl_tp4.txt 2>&1; cat gpurun_out/tps/tl_tp4.txt
A=HX_DEFER_QKV=0 B=HX_DEFER_QKV=1 bash tools/gpu_ab_dist.sh
cp gpurun_out/abd_tp4.log gpurun_out/abd_tp2.log gpurun_out/tps/ 2>/dev/null
