"""The deferred-QKV hand-off in isolation: hx_linear(defer_reduce) of the QKV
shard followed by hx_attn_decode_rope_append_sk, with hx_debug_trace: how long
after its dependency wait the attention has q gathered from the partial slots.

    python tools/def_gather_bench.py [tp]     (70B shard shapes, b = 32, ctx 1024)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2311_11514_b200 import ops

tp = int(next((a for a in sys.argv[1:] if a.isdigit()), 4))
b, H, hd, page, ctx = 32, 8192, 128, 64, 1024
hq, hkv = 64 // tp, 8 // tp
n = (hq + 2 * hkv) * hd
dev = "cuda"
lib = ops.load()
g = torch.Generator(device=dev).manual_seed(0)
w = ops.PackedWeight((torch.randn(n, H, device=dev, generator=g) * 0.02).bfloat16())
x = torch.randn(b, H, device=dev, generator=g).bfloat16()
lws = torch.zeros(ops.linear_workspace(torch.bfloat16, b, n, H) // 4 + 64, dtype=torch.int32, device=dev)
y = torch.empty(b, n, device=dev)
maxb = (ctx + 4 + page - 1) // page
kc = torch.zeros(b * maxb, hkv, page, hd, device=dev, dtype=torch.bfloat16)
vc = torch.zeros_like(kc)
bt = torch.arange(b * maxb, device=dev, dtype=torch.int32).view(b, maxb).contiguous()
sl = torch.full((b,), ctx, dtype=torch.int32, device=dev)
o = torch.empty(b, hq * hd, device=dev, dtype=torch.bfloat16)
aws = torch.zeros(ops.attn_decode_workspace(b, hq, hkv, hd, maxb * page) // 4 + 64, dtype=torch.int32, device=dev)


AGAIN = "--again" in sys.argv  # a second attention re-reading the same partials


GG = "--gemm-gemm" in sys.argv  # GEMM -> GEMM release only


def step():
    if GG:
        ops.linear(w, x, y, b, lws, defer_reduce=True)
        ops.linear(w, x, y, b, lws, defer_reduce=True)
        return
    ops.linear(w, x, y, b, lws, defer_reduce=True)
    ops.attn_decode_rope_append_sk(y, lws, H, kc, vc, bt, sl, o, b, hq, hkv, hd, maxb * page, 1e4, aws)
    if AGAIN:
        ops.attn_decode_rope_append_sk(y, lws, H, kc, vc, bt, sl, o, b, hq, hkv, hd, maxb * page, 1e4, aws)


step()
torch.cuda.synchronize()
cap = 64 * 1024
buf = torch.zeros(cap * 8, dtype=torch.int64, device=dev)
lib.hx_debug_trace(buf.data_ptr(), cap)
graph = torch.cuda.CUDAGraph()   # launched from a graph: the host never paces the GPU
with torch.cuda.graph(graph):
    for _ in range(4):
        step()
used = lib.hx_debug_trace(None, 0)
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
tr = buf.view(-1, 8)[:used].cpu().numpy().astype(np.int64)
att = (tr[:, 3] >> 40) & 1
G = 148
if GG:
    for k in range(used // (2 * G)):
        a, c = tr[2 * k * G:(2 * k + 1) * G], tr[(2 * k + 1) * G:(2 * k + 2) * G]
        print(f"GEMM -> GEMM: second GEMM's wait passed {(c[:, 1].min() - a[:, 2].max()) / 1e3:+.2f}..{(c[:, 1].max() - a[:, 2].max()) / 1e3:+.2f} us "
              f"after the first's end; first CTA start {(c[:, 0].min() - a[:, 2].max()) / 1e3:+.2f}")
    sys.exit(0)
i, k = 0, 0
while i < used:
    gm = tr[i:i + G]
    j = i + G
    a = j
    while a < used and att[a]:
        a += 1
    at = tr[j:a]
    if AGAIN:   # two launches back to back: split the run in half
        h = (a - j) // 2
        at2 = tr[j + h:a]
        at = tr[j:j + h]
        print(f"   second attention: wait->q ready med {np.median(at2[:, 4] - at2[:, 1]) / 1e3:.2f} us")
    end = gm[:, 2].max()
    us = lambda v: (v - end) / 1e3
    print(f"rep {k}: gemm run {(gm[:, 2].max() - gm[:, 1].min()) / 1e3:.2f} us; attention (rel. GEMM end): "
          f"wait {us(at[:, 1].min()):.2f}..{us(at[:, 1].max()):.2f}  q ready med {us(np.median(at[:, 4])):.2f} "
          f"max {us(at[:, 4].max()):.2f}  loop done max {us(at[:, 5].max()):.2f}  end {us(at[:, 2].max()):.2f}  "
          f"wait->q ready med {np.median(at[:, 4] - at[:, 1]) / 1e3:.2f}")
    i, k = a, k + 1
