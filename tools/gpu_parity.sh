#!/bin/bash
# Parity run on a 1-GPU box: collectives harness, smoke, engine parity (incl. C2 full depth).
# usage: gpurun --timeout 2400 -- bash tools/gpu_parity.sh [pytest -k expr]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${1:-}
timeout 600 python -m pytest tests/test_gpu_collectives.py -q -rf > gpurun_out/coll.log 2>&1; echo coll rc=$?; tail -3 gpurun_out/coll.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -5 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_engine.py -q -rf -s --durations=8 ${K:+-k "$K"} > gpurun_out/engine.log 2>&1; echo engine rc=$?; grep -E "C2|bf16 teacher|passed|failed|FAILED|^E " gpurun_out/engine.log | tail -30
