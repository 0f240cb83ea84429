cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_n2c.json 2> gpurun_out/bench_n2c.err; echo bench2 rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_n2c.json')); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], d['prefill_ms'], d['step_roofline']['frac'], r['frac'], d['e2e']['value'])"
