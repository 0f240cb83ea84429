"""Measured service time of one pipeline of a plan (the reference's
``service_times`` entry, simulate.py:135-142) on this box's GPUs.

    torchrun --nproc-per-node <pipeline GPUs> --master-addr 127.0.0.1 tools/measure_service.py \
        --plan plan.json --pipeline 0 --model llama2-70b --task 32,1024,256 --out svc_p0.json

The pipeline's stages keep their TP degrees and layer counts; its device ids
are renumbered 0..n-1 in stage order (every B200 of an NVSwitch node is
equivalent), so one pipeline of an 8-GPU plan is measured on n GPUs. Rank 0
writes ``{"replica", "batch_size", "input_len", "output_len", "seconds",
"prefill_s", "decode_s", "plan", "layers", "gpu_type"}`` -- an entry of the ``--service`` table of
``python -m paper_2311_11514_b200.planner simulate``.
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import torch.distributed as dist

from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.plan import GlobalAssignment, StageAssignment, TaskSpec, load_plan, plan_notation


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", required=True)
    ap.add_argument("--pipeline", type=int, default=0)
    ap.add_argument("--model", default="llama2-70b")
    ap.add_argument("--task", default="32,1024,256")
    ap.add_argument("--repeats", type=int, default=2)
    ap.add_argument("--gpu-type", default="b200", help="cluster GPU type id the measurement applies to")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    pipe = load_plan(a.plan).pipelines[a.pipeline]
    stages, d = [], 0
    for st in pipe:
        stages.append(StageAssignment(tuple(range(d, d + st.tp_degree)), st.num_layers))
        d += st.tp_degree
    sub = GlobalAssignment((tuple(stages),))
    task = TaskSpec(*[int(x) for x in a.task.split(",")])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != d:
        raise SystemExit(f"pipeline {plan_notation(pipe)} needs {d} ranks, have {world}")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = preset(a.model)
    n_layers = sum(st.num_layers for st in pipe)
    if n_layers != cfg.num_layers:   # one stage of a larger pipeline, measured on its own
        cfg = preset(a.model, num_layers=n_layers)
    eng = Engine(sub, cfg, dtype="bf16", batch=task.batch_size, max_prompt=task.input_len, max_out=task.output_len,
                 comm="dist" if world > 1 else "local", device=dev, weights="device")
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(task.batch_size, task.input_len), dtype=np.int32)
    eng.generate(prompt, task.output_len)   # warm-up + graph capture
    runs = [eng.generate(prompt, task.output_len) for _ in range(a.repeats)]
    vals = torch.tensor([[r.prefill_s + r.decode_s, r.prefill_s, r.decode_s] for r in runs], dtype=torch.float64,
                        device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    if (dist.get_rank() if world > 1 else 0) == 0:
        v = vals.cpu().numpy()
        doc = {"replica": a.pipeline, "batch_size": task.batch_size, "input_len": task.input_len,
               "output_len": task.output_len, "seconds": float(statistics.median(v[:, 0])),
               "prefill_s": float(statistics.median(v[:, 1])), "decode_s": float(statistics.median(v[:, 2])),
               "plan": plan_notation(pipe), "layers": [s.num_layers for s in pipe], "gpus": d,
               "gpu_type": a.gpu_type, "device_name": torch.cuda.get_device_name(dev),
               "model_layers": cfg.num_layers}
        Path(a.out).write_text(json.dumps(doc, indent=1) + "\n")
        print(json.dumps(doc), flush=True)
    if world > 1:
        dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
