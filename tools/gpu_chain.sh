#!/bin/bash
# kernel-boundary micro-benchmark + full-step GEMM timeline (launch lead)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/chain
./tools/micro/chain_latency > gpurun_out/chain/chain.txt 2>&1
python tools/gemm_timeline.py llama2-7b --full-step > gpurun_out/chain/tl7b.txt 2>&1
python tools/gemm_timeline.py llama2-70b --tp=4 --full-step > gpurun_out/chain/tl70tp4.txt 2>&1
cat gpurun_out/chain/chain.txt; tail -12 gpurun_out/chain/tl7b.txt; tail -12 gpurun_out/chain/tl70tp4.txt
