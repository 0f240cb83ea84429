"""Deferred split-K into the push all-reduce, in isolation on one GPU (TP=1
group: no peers, the same kernel): hx_linear(O shard) -> all-reduce(+norm) ->
hx_linear(gate/up shard), captured in a graph; the gate/up GEMM's wait after the
O GEMM's end (hx_debug_trace) with the O GEMM deferred or not.

    python tools/def_ar_bench.py [tp]    (70B shard shapes, b = 32)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2311_11514_b200 import ops

tp = int(next((a for a in sys.argv[1:] if a.isdigit()), 4))
b, H = 32, 8192
k_o, n_gu = 8192 // tp, 2 * 28672 // tp
dev = "cuda"
lib = ops.load()
g = torch.Generator(device=dev).manual_seed(0)
wo = ops.PackedWeight((torch.randn(H, k_o, device=dev, generator=g) * 0.02).bfloat16())
wgu = ops.PackedWeight((torch.randn(n_gu, H, device=dev, generator=g) * 0.02).bfloat16())
a = torch.randn(b, k_o, device=dev, generator=g).bfloat16()
ws_words = max(ops.linear_workspace(torch.bfloat16, b, H, k_o), ops.linear_workspace(torch.bfloat16, b, n_gu, H))
lws = torch.zeros(ws_words // 4 + 64, dtype=torch.int32, device=dev)
x = torch.zeros(b, H, device=dev)
gain = torch.ones(H, device=dev)
h = torch.empty(b, H, device=dev, dtype=torch.bfloat16)
gu = torch.empty(b, n_gu, device=dev)
grp = ops.PeerAllReduce.local_group(1, b, H, 4, mode="push", payload="bf16")[0]


def step(deferred):
    ops.linear(wo, a, grp.slot(0), b, lws, defer_reduce=deferred)
    kw = {"gemm_ws": lws, "k_dim": k_o} if deferred else {}
    grp.allreduce_residual_rmsnorm(x, 0, gain, h, b, 1e-5, **kw)
    ops.linear(wgu, h, gu, b, lws)


for deferred in (False, True):
    step(deferred)
    torch.cuda.synchronize()
    cap = 64 * 1024
    buf = torch.zeros(cap * 8, dtype=torch.int64, device=dev)
    lib.hx_debug_trace(buf.data_ptr(), cap)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(4):
            step(deferred)
    used = lib.hx_debug_trace(None, 0)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    tr = buf.view(-1, 8)[:used].cpu().numpy().astype(np.int64)
    G = 148
    rows = []
    for k in range(used // (2 * G)):
        o, q = tr[2 * k * G:(2 * k + 1) * G], tr[(2 * k + 1) * G:(2 * k + 2) * G]
        rows.append(((o[:, 2].max() - o[:, 1].min()) / 1e3, (q[:, 1].min() - o[:, 2].max()) / 1e3,
                     (q[:, 2].max() - o[:, 1].min()) / 1e3))
    r = np.median(np.array(rows[1:]), axis=0)
    print(f"tp={tp} O {'deferred' if deferred else 'fix-up  '}: O run {r[0]:6.2f} us, gate/up wait after O end "
          f"{r[1]:6.2f} us, O wait -> gate/up end {r[2]:6.2f} us")
grp.close()
