"""Decode-attention micro-benchmark (fused RoPE + KV append + paged GQA
attention, hx_attn_decode_rope_append) at the decode shapes of the configs.
L layer caches are cycled so the KV stream (> 126 MB L2) comes from HBM.

    python tools/attn_bench.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2311_11514_b200 import ops

SHAPES = {  # name: (batch, hq, hkv, ctx)
    "7b b8 ctx575": (8, 32, 32, 575),
    "70b tp1 b32 ctx1151": (32, 64, 8, 1151),
    "70b tp2 b32 ctx1151": (32, 32, 4, 1151),
    "70b tp4 b32 ctx1151": (32, 16, 2, 1151),
}


def bench(b, hq, hkv, ctx, L=8, reps=20):
    hd, page = 128, 64
    maxb = (ctx + 1 + page - 1) // page + 1
    nb = b * maxb
    dev = "cuda"
    kc = torch.randn(L, nb, hkv, page, hd, device=dev).bfloat16()
    vc = torch.randn(L, nb, hkv, page, hd, device=dev).bfloat16()
    bt = torch.randperm(nb, device=dev, dtype=torch.int32).view(b, maxb).contiguous()
    sl = torch.full((b,), ctx - 1, dtype=torch.int32, device=dev)
    qkv = torch.randn(b, (hq + 2 * hkv) * hd, device=dev).bfloat16()
    o = torch.empty(b, hq * hd, device=dev).bfloat16()
    wsb = ops.attn_decode_workspace(b, hq, hkv, hd, maxb * page)
    ws = torch.zeros(max(wsb, 256) // 4 + 64, dtype=torch.int32, device=dev)

    def run():
        for l in range(L):
            ops.attn_decode_rope_append(qkv, kc[l], vc[l], bt, sl, o, b, hq, hkv, hd, maxb * page, 1e4, ws)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    g.replay()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(reps):
        g.replay()
    s1.record()
    torch.cuda.synchronize()
    us = s0.elapsed_time(s1) / reps / L * 1e3
    nbytes = b * ctx * 2 * hkv * hd * 2
    return us, nbytes / us / 1e3


def main():
    ops.load()
    for name, shp in SHAPES.items():
        us, gbs = bench(*shp)
        print(f"{name:22s} ctas={os.environ.get('HX_ATTN_CTAS', '296'):>4s}: {us:7.2f} us/layer  "
              f"{gbs:7.1f} GB/s ({gbs / 6551:.2f} of 6551)", flush=True)


if __name__ == "__main__":
    main()
