#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/apw
for v in 3 0 1; do
  echo "== HX_ATTN_PREWAIT=$v"
  HX_ATTN_PREWAIT=$v python tools/attn_timeline.py llama2-70b --tp=4 2>&1 | grep -E "wait done max|q ready|loop done|combine|attn end|O wait|O end|CTAs with"
  HX_ATTN_PREWAIT=$v python tools/attn_timeline.py llama2-7b 2>&1 | grep -E "q ready med|attn end|O wait|O end"
done 2>&1 | tee gpurun_out/apw/tl.txt
