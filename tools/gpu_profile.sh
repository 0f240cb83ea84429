#!/bin/bash
# Decode-GEMM evidence on a 1-GPU box: per-CTA timelines of the decode step (7B, 70B TP=4 shard, 13B TP=2
# shard) and ncu --set full of one launch per GEMM shape (DRAM traffic vs algorithmic bytes).
# usage: gpurun --timeout 2400 -- bash tools/gpu_profile.sh [timeline] [traffic]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WHAT=${@:-timeline traffic}
for w in $WHAT; do case $w in
  timeline)
    timeout 300 python tools/gemm_timeline.py llama2-7b --full-step > gpurun_out/tl_7b.txt 2>&1; echo "tl 7b rc=$?"; tail -6 gpurun_out/tl_7b.txt
    timeout 300 python tools/gemm_timeline.py llama2-70b --tp=4 --layers=20 --full-step > gpurun_out/tl_70b_tp4.txt 2>&1; echo "tl 70b tp4 rc=$?"; tail -6 gpurun_out/tl_70b_tp4.txt
    timeout 300 python tools/gemm_timeline.py llama2-13b --tp=2 --full-step > gpurun_out/tl_13b_tp2.txt 2>&1; echo "tl 13b tp2 rc=$?"; tail -6 gpurun_out/tl_13b_tp2.txt ;;
  traffic) bash tools/gemm_traffic.sh ;;
esac; done
