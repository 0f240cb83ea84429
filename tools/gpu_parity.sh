cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_collectives.py -q -rf -x > gpurun_out/coll.log 2>&1; echo coll rc=$?; tail -3 gpurun_out/coll.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_engine.py -q -rf -s --durations=15 > gpurun_out/engine.log 2>&1; echo engine rc=$?; grep -E "bf16 teacher|passed|failed|FAILED" gpurun_out/engine.log | tail -30
