cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "decode/" -k regex:"attn_decode_mma|sk_residual" -s 2 -c 2 --set full --import-source on --clock-control none -o gpurun_out/attn_full python tools/profile_decode.py > gpurun_out/ncu8.log 2>&1
echo ncu rc=$?
