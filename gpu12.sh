cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "passed|failed|Error|error|assert" | tail -20
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench rc=$?
cat gpurun_out/bench6.json; tail -3 gpurun_out/bench6.err
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_decode4.csv python tools/profile_decode.py > gpurun_out/ncu5.log 2>&1
echo ncu rc=$?
