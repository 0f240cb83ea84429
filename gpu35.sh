cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python tools/profile_decode.py > gpurun_out/ncu_l.log 2>&1
echo launches rc=$?
timeout 900 ncu --nvtx --nvtx-include "decode/" -k regex:"gemm_streamk|attn_decode_tma|sk_residual" -s 3 -c 4 --set full --import-source on --clock-control none -o gpurun_out/r01_full python tools/profile_decode.py > gpurun_out/ncu_f.log 2>&1
echo full rc=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 600 --csv --log-file gpurun_out/bench_launches_r01.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
echo bench-ncu rc=$?
