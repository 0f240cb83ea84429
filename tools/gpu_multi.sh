#!/bin/bash
# Multi-GPU checks on a gpurun --gpus 4 box: NCCL/NVLink tests, C3 (13B [2,1] vs [2,2]) and 70B bench lines.
# usage: gpurun --gpus 4 --timeout 2400 -- bash tools/gpu_multi.sh [what...]   (what: tests c3 70b; default all)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WHAT=${@:-tests c3 70b}
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
run() {  # run <tag> <nproc> <bench args...>
  local tag=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
  echo "$tag rc=$?"; tail -1 gpurun_out/bench_$tag.json | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); s=d['step_roofline']
  print(' ', d['config']['workload'], 'value', d['value'], 'p50', d['p50_decode_step_ms'], 'T*', s['t_star_ms'], 'frac', s['frac'], 'prefill_ms', d['prefill_ms'], 'e2e', d['e2e']['value'])
except Exception as e: print('  parse fail', e)"
}
for w in $WHAT; do case $w in
  tests) timeout 1200 python -m pytest tests/test_dist.py -m gpu -q -rs > gpurun_out/dist_gpu.log 2>&1; echo "dist tests rc=$?"; tail -3 gpurun_out/dist_gpu.log ;;
  c3) run c3asym 3 --workload c3-asym --steps 5 --warmup 3; run c3sym 4 --workload c3-sym --steps 5 --warmup 3 ;;
  70b) run n2 2 --steps 2 --warmup 3; run n4 4 --steps 2 --warmup 3 ;;
esac; done
