cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full4.log 2>&1; echo rc=$?; tail -1 gpurun_out/pytest_full4.log; grep -E "^FAILED|Error" gpurun_out/pytest_full4.log | head -8
for e in "1 1" "0 0" "1 0" "0 1"; do set -- $e
  echo "swiglu=$1 rope=$2"; HX_FUSE_SWIGLU=$1 HX_FUSE_ROPE=$2 timeout 600 python tools/ablate_step.py 2>&1 | grep -E "^none|all-but"
done
for e in "1 1" "0 0"; do set -- $e
HX_FUSE_SWIGLU=$1 HX_FUSE_ROPE=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b15.json 2>/dev/null
tail -1 gpurun_out/b15.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], d['prefill_ms'], r['gemm_ms_per_step'], d['e2e']['value'])"
done
