"""Decode-step ablation (timing only; outputs are garbage when ops are skipped):
the 7B b=8 decode step replayed as the engine's CUDA graph with one class of
kernels turned into no-ops, to attribute the step time.

    python tools/ablate_step.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

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


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    cfg = preset(model)
    b, s_in, s_out = 8, 512, 48
    groups = {
        "none": [],
        "attention": ["attn_decode"],
        "rope+append": ["rope_kv_append"],
        "swiglu": ["swiglu"],
        "norms": ["splitk_residual_rmsnorm", "residual_add_rmsnorm", "rmsnorm"],
        "gemms": ["linear"],
        "all-but-gemm": ["attn_decode", "rope_kv_append", "swiglu", "splitk_residual_rmsnorm",
                         "residual_add_rmsnorm", "rmsnorm"],
    }
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(b, s_in), dtype=np.int32)
    eng = Engine(simple_plan([1], [cfg.num_layers]), cfg, dtype="bf16", batch=b, max_prompt=s_in, max_out=s_out,
                 device="cuda:0", weights="device")
    base = {}
    for name, skip in groups.items():
        px = Proxy(skip)
        for e in eng.execs:
            e.k = px
        eng._graphs = None  # recapture with this op set
        eng.generate(prompt, s_out)
        r = eng.generate(prompt, s_out)
        base[name] = float(np.median(r.step_ms))
        print(f"{name:14s} skip={skip}: p50 decode step {base[name]:.3f} ms "
              f"(saves {base.get('none', base[name]) - base[name]:.3f} ms)", flush=True)


if __name__ == "__main__":
    main()
