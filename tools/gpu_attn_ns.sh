#!/bin/bash
# decode attention ring-depth / CTAs-per-SM A/B (HX_ATTN_NS: default 3-deep x 2 CTAs/SM, 2 = 2-deep x 3 CTAs/SM)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ans
for v in 0 2 0 2; do
  echo "HX_ATTN_NS=$v"; HX_ATTN_NS=$v python tools/attn_bench.py
done 2>&1 | tee gpurun_out/ans/attn.txt
for v in 0 2; do
  HX_ATTN_NS=$v python tools/gemm_timeline.py llama2-70b --tp=4 --full-step > gpurun_out/ans/tl70tp4_$v.txt 2>&1
  echo "NS=$v tp4: $(grep 'mean o ' gpurun_out/ans/tl70tp4_$v.txt)"
  HX_ATTN_NS=$v python tools/gemm_timeline.py llama2-7b --full-step > gpurun_out/ans/tl7b_$v.txt 2>&1
  echo "NS=$v 7b: $(grep 'mean o ' gpurun_out/ans/tl7b_$v.txt) $(grep total gpurun_out/ans/tl7b_$v.txt)"
done
HX_ATTN_NS=2 timeout 600 python -m pytest tests -q -m gpu -x -k "attn or decode" 2>&1 | tail -3
