cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full2.log 2>&1; echo rc=$?; tail -1 gpurun_out/pytest_full2.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench rc=$?
tail -1 gpurun_out/bench_r1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], d['prefill_ms'], d['step_roofline']['frac'], r['frac'], d['e2e']['value'], d['cpu_baseline'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref rc=$?; tail -1 gpurun_out/bench_ref.json | cut -c1-300
