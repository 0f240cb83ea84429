#!/bin/bash
# Round profile evidence for the 7B N=1 bench workload (1 GPU):
#   launch list of one decode step (NVTX range) and of the bench command,
#   ncu --set full of the decode GEMM (top kernel) and the decode attention.
# usage: gpurun --timeout 1500 -- bash tools/profile_round.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_decode.py > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/decode_step_launches.csv python tools/profile_decode.py > /dev/null 2>&1; echo "step list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 800 --csv \
  --log-file gpurun_out/bench_cmd_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "bench list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_streamk -s 200 -c 4 \
  -o gpurun_out/prof_gemm python tools/profile_decode.py > /dev/null 2>&1; echo "gemm full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode_tma -s 40 -c 2 \
  -o gpurun_out/prof_attn python tools/profile_decode.py > /dev/null 2>&1; echo "attn full rc=$?"
