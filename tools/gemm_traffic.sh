#!/bin/bash
# ncu --set full of one decode-GEMM launch per shape (tools/gemm_traffic.py). The reports are reduced to
# raw-page CSVs on the box (gpurun_out/traffic/<shape>.csv); only the first shape's .ncu-rep is kept.
# usage: gpurun --timeout 1800 -- bash tools/gemm_traffic.sh [shape ...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/traffic
SH=${@:-$(python tools/gemm_traffic.py shapes)}
keep=1
for s in $SH; do
  timeout 300 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "measure/" \
    -k regex:gemm_streamk -o /tmp/tr_$s python tools/gemm_traffic.py run $s > gpurun_out/traffic/$s.log 2>&1
  echo "$s rc=$?"
  ncu -i /tmp/tr_$s.ncu-rep --page raw --csv > gpurun_out/traffic/$s.csv 2>/dev/null
  if [ $keep = 1 ]; then cp /tmp/tr_$s.ncu-rep gpurun_out/traffic/; keep=0; fi
  rm -f /tmp/tr_$s.ncu-rep
done
