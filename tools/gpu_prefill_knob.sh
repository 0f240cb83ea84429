#!/bin/bash
# same-box A/B of HX_GEMM_PERSISTENT (1: >= 4096 rows only, 2: also micro-batches) on micro-batched prefills
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pfk
for v in 1 3 2 1 3 2; do
  for spec in "n2 2" "c3asym 3 --workload c3-asym"; do
    set -- $spec; tag=$1; n=$2; shift 2
    HX_GEMM_PERSISTENT=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n --steps 2 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/pfk/$tag.json 2> gpurun_out/pfk/$tag.err
    echo "HX_GEMM_PERSISTENT=$v $tag: $(tail -1 gpurun_out/pfk/$tag.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill_ms', d['prefill_ms'], 'e2e', d['e2e']['value'])")"
  done
done
