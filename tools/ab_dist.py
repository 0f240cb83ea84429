"""A/B of two engine settings on the same GPUs, interleaved to cancel drift
(torchrun, one rank per GPU; a single-stage plan [tp] over a --layers-deep
copy of the model).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ab_dist.py --tp 2 --layers 40 \
        --a HX_AR_PAYLOAD=fp32 --b HX_AR_PAYLOAD=bf16

Environment assignments in --a / --b (comma-separated) are applied while that
engine is constructed (the engine reads its switches at construction).
With --tp 1 it runs in one process (no torchrun needed).
"""
import argparse
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
from paper_2311_11514_b200.plan import simple_plan


def build(spec, a, cfg, dev, comm):
    saved = {}
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=", 1)
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        return Engine(simple_plan([a.tp], [a.layers]), cfg, dtype="bf16", batch=a.batch, max_prompt=a.s_in,
                      max_out=a.s_out, comm=comm, device=dev, weights="device")
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-70b")
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--s-in", type=int, default=1024)
    ap.add_argument("--s-out", type=int, default=33)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--a", default="")
    ap.add_argument("--b", default="")
    a = ap.parse_args()
    if a.tp > 1:
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
        comm, rank = "dist", dist.get_rank()
    else:
        dev, comm, rank = torch.device("cuda", 0), "local", 0
    cfg = preset(a.model, num_layers=a.layers)
    engs = {"A": build(a.a, a, cfg, dev, comm), "B": build(a.b, a, cfg, dev, comm)}
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(a.batch, a.s_in), dtype=np.int32)
    steps = {k: [] for k in engs}
    for k, e in engs.items():
        e.generate(prompt, a.s_out)
    for _ in range(a.rounds):
        for k, e in engs.items():
            steps[k] += e.generate(prompt, a.s_out).step_ms
    if rank == 0:
        for k, spec in (("A", a.a), ("B", a.b)):
            print(f"{k} [{spec or 'default'}]: p50 decode step {statistics.median(steps[k]):.3f} ms "
                  f"(p10 {np.percentile(steps[k], 10):.3f}, p90 {np.percentile(steps[k], 90):.3f}, n={len(steps[k])})",
                  flush=True)
    if a.tp > 1:
        dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
