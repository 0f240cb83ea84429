cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_decode.csv python tools/profile_decode.py > gpurun_out/ncu1.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu1.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
cat gpurun_out/bench2.json; tail -5 gpurun_out/bench2.err
