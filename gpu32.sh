cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist.py -m gpu -q -rf > gpurun_out/pytest_dist4.log 2>&1; echo rc=$?
tail -2 gpurun_out/pytest_dist4.log; grep -E "FAILED" gpurun_out/pytest_dist4.log | head -5
for p in 1 0; do
HX_PEER_AR=$p timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$p bench.py --gpus 4 --steps 2 --warmup 3 > gpurun_out/bench_n4_p$p.json 2> gpurun_out/bench_n4_p$p.err; echo bench4 peer=$p rc=$?
tail -1 gpurun_out/bench_n4_p$p.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('peer',$p, d['value'], d['p50_decode_step_ms'], d['prefill_ms'], d['step_roofline']['frac'], r['frac'], d['e2e']['value'])"
done
