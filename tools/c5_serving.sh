#!/bin/bash
# C5 on a 4-GPU box: GA plan with the restated planner (same plan as the
# reference), then measured service times of every distinct pipeline shape.
# usage: gpurun --gpus 4 --timeout 3000 -- bash tools/c5_serving.sh
cd $GRAFT_REPO_ROOT
B=tests/golden/planner/b200_422/inputs
mkdir -p gpurun_out/c5/svc
python -m paper_2311_11514_b200.planner plan --cluster $B/cluster.json --model $B/model.json --workload $B/workload.json \
  --slo $B/slo.json --out-dir gpurun_out/c5/ga --pop 16 --gens 30 --seed 0 | tail -2
cmp gpurun_out/c5/ga/plan.json tests/golden/planner/b200_422/plan_s0/plan.json && echo "GA plan identical to the reference's"
# pipelines 0-2: the GA plan's and the homogeneous layouts' shapes (<= 4 GPUs, measured whole);
# 3-4: the single stages of the 8-GPU [4,2,2] 40/20/20 pipeline (its service time is composed from them)
cat > gpurun_out/c5/shapes.json <<'J'
{"schema_version": 1, "pipelines": [
 {"stages": [{"devices": [0, 1], "layers": 40}, {"devices": [2, 3], "layers": 40}]},
 {"stages": [{"devices": [0, 1], "layers": 80}]},
 {"stages": [{"devices": [0, 1, 2, 3], "layers": 80}]},
 {"stages": [{"devices": [0, 1, 2, 3], "layers": 40}]},
 {"stages": [{"devices": [0, 1], "layers": 20}]}]}
J
i=0
for k_n in 0:4 1:2 2:4 3:4 4:2; do k=${k_n%%:*}; n=${k_n##*:}
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + k)) \
    tools/measure_service.py --plan gpurun_out/c5/shapes.json --pipeline $k --out gpurun_out/c5/svc/p$k.json 2>&1 | grep -E '^\{|Error' | head -3
done
python tools/c5_report.py --plan gpurun_out/c5/ga/plan.json --svc gpurun_out/c5/svc --out gpurun_out/c5/c5_serving.json > /dev/null && echo report ok
