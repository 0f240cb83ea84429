cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -s 2>&1 | grep -E "passed|failed|Error|error|bf16 teacher|assert" | tail -20
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_decode2.csv python tools/profile_decode.py > gpurun_out/ncu2.log 2>&1
echo ncu rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench rc=$?
cat gpurun_out/bench3.json; tail -5 gpurun_out/bench3.err
