"""Decode-step ablation of one TP stage under torch.distributed (timing only;
outputs are garbage when ops are skipped).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ablate_dist.py --tp 2 --layers 40

Builds a single-stage plan [tp] over a ``--layers``-deep copy of the model and
replays its decode graph with one class of kernels turned into no-ops.
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

from paper_2311_11514_b200 import ops
from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.plan import simple_plan


class Proxy:
    def __init__(self, skip):
        self.skip = set(skip)

    def __getattr__(self, name):
        if name in self.skip:
            return lambda *a, **k: None
        return getattr(ops, name)


class ParProxy:
    def __init__(self, par, skip):
        self.par, self.skip = par, skip

    def slot(self, site):
        return self.par.slot(site)

    def allreduce_residual_rmsnorm(self, *a, **k):
        if not self.skip:
            self.par.allreduce_residual_rmsnorm(*a, **k)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama2-70b")
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--s-in", type=int, default=1024)
    a = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = preset(a.model, num_layers=a.layers)
    eng = Engine(simple_plan([a.tp], [a.layers]), cfg, dtype="bf16", batch=a.batch, max_prompt=a.s_in, max_out=16,
                 comm="dist", device=dev, weights="device")
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(a.batch, a.s_in), dtype=np.int32)
    groups = {
        "none": ([], False),
        "peer-allreduce": ([], True),
        "attention": (["attn_decode_rope_append", "attn_decode"], False),
        "swiglu": (["swiglu"], False),
        "gemms": (["linear"], False),
        "all-but-gemm": (["attn_decode_rope_append", "attn_decode", "swiglu", "rmsnorm",
                          "residual_add_rmsnorm", "splitk_residual_rmsnorm"], True),
    }
    pars = [e.par for e in eng.execs]
    for name, (skip, skip_ar) in groups.items():
        for e, par in zip(eng.execs, pars):
            e.k = Proxy(skip)
            if par is not None:
                e.par = ParProxy(par, skip_ar)
        eng._graphs = None
        eng.generate(prompt, 16)
        r = eng.generate(prompt, 16)
        if dist.get_rank() == 0:
            print(f"{name:15s}: p50 decode step {statistics.median(r.step_ms):.3f} ms", flush=True)
    dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
