cd $GRAFT_REPO_ROOT
for cfg in "1 4" "1 6" "1 8" "1 10" "1 12" "2 6"; do set -- $cfg
HX_SK_CTAS=$1 HX_SK_STAGES=$2 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_$1_$2.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b_$1_$2.json')); r=d['roofline']; print('ctas',$1,'stages',$2, d['value'], d['p50_decode_step_ms'], r['gemm_ms_per_step'], {k:v['GBps'] for k,v in r['per_shape'].items()})"
done
