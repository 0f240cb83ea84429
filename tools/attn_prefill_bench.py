"""Prefill (causal, paged) attention throughput at the configs' shapes.

    python tools/attn_prefill_bench.py      # HX_PF_WARPS=4|8 selects the CTA shape
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2311_11514_b200 import ops

SHAPES = {"7b b8 s512": (8, 512, 32, 32), "70b-tp1 mb4 s1024": (4, 1024, 64, 8), "70b-tp2 mb4 s1024": (4, 1024, 32, 4)}


def main():
    ops.load()
    hd, page = 128, 64
    for name, (b, s, hq, hkv) in SHAPES.items():
        maxb = (s + page - 1) // page
        nb = b * maxb
        kc = torch.randn(nb, hkv, page, hd, device="cuda").bfloat16()
        vc = torch.randn(nb, hkv, page, hd, device="cuda").bfloat16()
        bt = torch.randperm(nb, device="cuda", dtype=torch.int32).view(b, maxb).contiguous()
        sl = torch.zeros(b, dtype=torch.int32, device="cuda")
        q = torch.randn(b * s, hq * hd, device="cuda").bfloat16()
        o = torch.empty_like(q)
        qkv = torch.randn(b * s, (hq + 2 * hkv) * hd, device="cuda").bfloat16()
        vt = torch.empty(b * hkv * hd * s, device="cuda").bfloat16()
        runs = {"mma.sync": lambda: ops.attn_prefill(q, kc, vc, bt, sl, o, b, s, hq, hkv, hd),
                "tcgen05": lambda: ops.attn_prefill_tc(q, kc, vt, bt, o, b, s, hq, hkv, hd),
                "tcgen05+vt": lambda: (ops.prefill_vt(qkv, vt, b, s, hq, hkv, hd),
                                       ops.attn_prefill_tc(q, kc, vt, bt, o, b, s, hq, hkv, hd))}
        for kind, fn in runs.items():
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 10 / 1e3
            flops = 4 * b * s * s * hq * hd / 2
            print(f"{name:20s} {kind:11s}: {t * 1e6:8.1f} us  {flops / t / 1e12:6.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
