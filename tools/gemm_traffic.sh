#!/bin/bash
# ncu --set full of one decode-GEMM launch per shape (tools/gemm_traffic.py) -> gpurun_out/traffic/<shape>.ncu-rep
# usage: gpurun --timeout 1800 -- bash tools/gemm_traffic.sh [shape ...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/traffic
SH=${@:-$(python tools/gemm_traffic.py shapes)}
for s in $SH; do
  timeout 300 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "measure/" \
    -k regex:gemm_streamk -o gpurun_out/traffic/$s python tools/gemm_traffic.py run $s > gpurun_out/traffic/$s.log 2>&1
  echo "$s rc=$?"
done
