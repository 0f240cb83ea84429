cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "decode/" -k regex:gemm_streamk -s 2 -c 1 --set full --import-source on --clock-control none -o gpurun_out/gemm_sk_full python tools/profile_decode.py > gpurun_out/ncu4.log 2>&1
echo ncu rc=$?; tail -3 gpurun_out/ncu4.log
