#!/bin/bash
# deferred split-K in the push all-reduce: kernel parity (1 GPU emulation), engine dist tests, TP stage A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/dar
timeout 900 python -m pytest tests/test_gpu_collectives.py tests/test_dist.py -q -x 2>&1 | tail -3 | tee gpurun_out/dar/tests.txt
A=HX_DEFER_AR=0 B=HX_DEFER_AR=1 bash tools/gpu_ab_dist.sh
TPS=4 timeout 600 bash tools/gpu_stage_tl.sh
