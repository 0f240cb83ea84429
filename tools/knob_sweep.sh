#!/bin/bash
# C-side knobs (read once at library load) need one process per setting:
# each line runs tools/ab_dist.py with the knob in the process environment
# (both A/B arms identical), baseline first and last to expose drift.
# usage: gpurun --gpus 4 --timeout 2400 -- bash tools/knob_sweep.sh
cd $GRAFT_REPO_ROOT
tp4() { env $1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port $((29500 + RANDOM % 400)) tools/ab_dist.py --tp 4 --layers 40 --rounds 2 2>&1 | grep -E "^A " | sed "s/^A \[default\]/tp4 $1/"; }
b7() { env $1 timeout 600 python tools/ab_dist.py --model llama2-7b --tp 1 --layers 32 --batch 8 --s-in 512 --rounds 2 \
  2>&1 | grep -E "^A " | sed "s/^A \[default\]/7b $1/"; }
for k in HX_NONE=0 HX_PDL=0 HX_SK_CTAS=296 HX_GEMM_L2PF=0 HX_GEMM_L2PF=48 HX_ATTN_NS=6 HX_ATTN_CLUSTER=0 HX_NONE=1; do tp4 $k; done
for k in HX_NONE=0 HX_PDL=0 HX_SK_CTAS=296 HX_GEMM_L2PF_ALL=1 HX_ATTN_NS=6 HX_NONE=1; do b7 $k; done
