"""Per-kernel cost of a PDL chain inside a CUDA graph: N back-to-back tiny
hx kernels (swiglu on one row), with PDL on and off. Bounds the fixed cost
of a kernel boundary in the decode step.

    python tools/launch_latency.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2311_11514_b200 import ops


def run(n=400, pdl=True, rows=1, inter=64):
    lib = ops.load()
    lib.hx_set_pdl(1 if pdl else 0)
    gu = torch.randn(rows, 2 * inter, device="cuda").bfloat16()
    a = torch.empty(rows, inter, device="cuda").bfloat16()
    ops.swiglu(gu, a, rows)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            ops.swiglu(gu, a, rows)
    g.replay()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(5):
        g.replay()
    s1.record()
    torch.cuda.synchronize()
    lib.hx_set_pdl(1)
    return s0.elapsed_time(s1) / 5 / n * 1e3


if __name__ == "__main__":
    for pdl in (True, False):
        for rows, inter in ((1, 64), (32, 14336)):
            print(f"pdl={pdl} swiglu rows={rows} inter={inter}: {run(pdl=pdl, rows=rows, inter=inter):.2f} us/kernel",
                  flush=True)
