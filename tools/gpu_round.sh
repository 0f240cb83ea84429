#!/bin/bash
# Round evidence on a 4-GPU box: full GPU test suite, smoke, N=1 bench (+ reference arm), multi-GPU bench
# lines (70B N=2/4, C3 13B [2,1] / [2,2]), ncu launch lists and --set full of the decode GEMM / attention.
# usage: gpurun --gpus 4 --timeout 3600 -- bash tools/gpu_round.sh [tests] [bench] [multi] [ncu]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/round
O=gpurun_out/round
WHAT=${@:-tests bench multi ncu}
for w in $WHAT; do case $w in
  tests)
    timeout 1500 python -m pytest tests -m gpu -q -rfs --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest_gpu.log | grep -E "passed|failed|FAILED|SKIP"
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log ;;
  bench)
    timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err; echo "ref rc=$?"; tail -1 $O/bench_ref_n1.json | cut -c1-300
    timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench n1 rc=$?"
    tail -1 $O/bench_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('N=1', d['value'], 'p50', d['p50_decode_step_ms'], 'frac', d['step_roofline']['frac'], 'gemm frac', r['frac'], 'prefill', d['prefill_ms'], 'e2e', d['e2e']['value'], 'clk', d['clocks'])" ;;
  multi)
    for spec in "n2 2" "n4 4" "c3asym 3 --workload c3-asym" "c3sym 4 --workload c3-sym"; do
      set -- $spec; tag=$1; n=$2; shift 2
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n --steps 5 --warmup 3 "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err
      echo "$tag rc=$?"; tail -1 $O/bench_$tag.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['step_roofline']
print(' ', d['config']['workload'], 'value', d['value'], 'p50', d['p50_decode_step_ms'], 'T*', s['t_star_ms'], 'frac', s['frac'], 'prefill_ms', d['prefill_ms'], 'e2e', d['e2e']['value'])"
    done ;;
  ncu)
    timeout 300 python tools/profile_decode.py > $O/plain.log 2>&1 || echo "profile_decode failed"
    timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/decode_step_launches.csv python tools/profile_decode.py > /dev/null 2>&1; echo "step list rc=$?"
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 800 --csv \
      --log-file $O/bench_cmd_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "bench list rc=$?"
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_streamk -s 200 -c 4 \
      -o $O/prof_gemm python tools/profile_decode.py > /dev/null 2>&1; echo "gemm full rc=$?"
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode_tma -s 40 -c 2 \
      -o $O/prof_attn python tools/profile_decode.py > /dev/null 2>&1; echo "attn full rc=$?"
    for r in prof_gemm prof_attn; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null; done
    du -sh $O ;;
esac; done
