set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L
timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q -k "linear_bf16 and 12288" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
