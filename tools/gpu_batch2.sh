#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/b2
O=gpurun_out/b2
timeout 900 python -m pytest tests/test_gpu_collectives.py tests/test_gpu_engine.py tests/test_dist.py -m gpu -q -rfs -k "credit or smaller_batch or nccl or tiny or gqa" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -4 $O/tests.log
for v in 0 1; do
  for spec in "n4 4" "c3asym 3 --workload c3-asym"; do
    set -- $spec; tag=$1; n=$2; shift 2
    HX_P2P_PREFILL=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline "$@" > $O/bench_${tag}_pf$v.json 2> $O/bench_${tag}_pf$v.err
    echo "$tag HX_P2P_PREFILL=$v rc=$? $(tail -1 $O/bench_${tag}_pf$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill_ms', d['prefill_ms'], 'value', d['value'], 'e2e', d['e2e']['value'])")"
  done
done
bash tools/gpu_sanitize.sh
