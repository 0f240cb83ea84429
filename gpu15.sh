cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L | wc -l
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf -k linear 2>&1 | grep -E "FAILED|passed|failed" | tail -3; done
timeout 900 python -m pytest tests/test_dist.py -m gpu -q -x -rf 2>&1 | grep -E "FAILED|passed|failed" | tail -5
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_n2b.json 2> gpurun_out/bench_n2b.err; echo bench2 rc=$?
cat gpurun_out/bench_n2b.json; grep -v "^W1018\|OMP\|\*\*\*" gpurun_out/bench_n2b.err | tail -5
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 2 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo bench4 rc=$?
cat gpurun_out/bench_n4.json; grep -v "^W1018\|OMP\|\*\*\*" gpurun_out/bench_n4.err | tail -5
