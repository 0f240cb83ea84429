"""Prefill GEMM throughput (hx_linear, n_tok > 64 path) at the configs' shapes, TFLOP/s."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2311_11514_b200 import ops

SHAPES = {  # (tokens, n_out, k)
    "7b qkv b8x512": (4096, 12288, 4096), "7b gate_up": (4096, 22016, 4096), "7b down": (4096, 4096, 11008),
    "70b-tp1 gate_up b32x1024": (32768, 57344, 8192), "70b-tp1 qkv": (32768, 10240, 8192),
    "70b-tp1 down": (32768, 8192, 28672), "70b-tp2 gate_up": (32768, 28672, 8192),
    # the engine's 70B prefill micro-batch (2048 token rows, bench N=2/4/8 plans)
    "70b mb tp1 gate_up": (2048, 57344, 8192), "70b mb tp1 qkv": (2048, 10240, 8192),
    "70b mb tp1 down": (2048, 8192, 28672), "70b mb tp2 gate_up": (2048, 28672, 8192),
    "70b mb tp4 gate_up": (2048, 14336, 8192), "70b mb tp4 qkv": (2048, 2560, 8192),
    "13b tp2 gate_up b8x512": (4096, 13824, 5120), "13b tp1 gate_up": (4096, 27648, 5120),
}
if len(sys.argv) > 1:
    SHAPES = {k: v for k, v in SHAPES.items() if any(a in k for a in sys.argv[1:])}
for name, (m, n, k) in SHAPES.items():
    w = ops.PackedWeight((torch.randn(n, k, device="cuda") * 0.02).bfloat16())
    x = torch.randn(m, k, device="cuda").bfloat16()
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        ops.linear(w, x, y, m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        ops.linear(w, x, y, m)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    print(f"{name:28s} {m}x{n}x{k}: {t * 1e3:8.3f} ms  {2 * m * n * k / t / 1e12:7.1f} TFLOP/s")
    del w, x, y
