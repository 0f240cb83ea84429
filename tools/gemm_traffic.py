"""DRAM traffic of the decode GEMM (hx_linear, stream-K tcgen05) per projection
shape, for the roofline.traffic field and the 70B shard evidence.

    python tools/gemm_traffic.py run <shape>      # one shape: 3 warm launches + 1 in NVTX range "measure"
    python tools/gemm_traffic.py shapes           # list shape names
    bash tools/gemm_traffic.sh                    # ncu --set full of every shape -> gpurun_out/traffic/

Each shape runs alone in its own process, so an ncu capture of the range
"measure/" holds exactly one launch of exactly that GEMM (no label mix-ups).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

# name -> (n_tok, n_out, k): the decode GEMMs of the bench workloads
SHAPES = {
    "7b_qkv": (8, 12288, 4096), "7b_o": (8, 4096, 4096), "7b_gate_up": (8, 22016, 4096),
    "7b_down": (8, 4096, 11008), "7b_lm_head": (8, 32000, 4096),
    "70b_tp4_qkv": (32, 2560, 8192), "70b_tp4_o": (32, 8192, 2048), "70b_tp4_gate_up": (32, 14336, 8192),
    "70b_tp4_down": (32, 8192, 7168),
    "70b_tp2_qkv": (32, 5120, 8192), "70b_tp2_o": (32, 8192, 4096), "70b_tp2_gate_up": (32, 28672, 8192),
    "70b_tp2_down": (32, 8192, 14336), "70b_tp2_lm_head": (32, 16000, 8192),
    "13b_tp2_qkv": (8, 7680, 5120), "13b_tp2_gate_up": (8, 13824, 5120), "13b_tp2_down": (8, 5120, 6912),
}


def algorithmic_bytes(n_tok, n_out, k, ybytes=4):
    return n_out * k * 2 + n_tok * k * 2 + n_tok * n_out * ybytes


def run(name):
    import torch
    from paper_2311_11514_b200 import ops
    n_tok, n_out, k = SHAPES[name]
    ops.load()
    g = torch.Generator(device="cuda").manual_seed(1)
    w = ops.PackedWeight((torch.randn(n_out, k, device="cuda", generator=g) * 0.02).bfloat16())
    x = torch.randn(n_tok, k, device="cuda", generator=g).bfloat16()
    y = torch.empty(n_tok, n_out, device="cuda", dtype=torch.float32)
    ws = torch.zeros(ops.linear_workspace(torch.bfloat16, n_tok, n_out, k) // 4 + 64, dtype=torch.int32,
                     device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ops.linear(w, x, y, n_tok, ws)
    flush.zero_()                 # the weights leave L2 (126 MB) like in the decode step
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("measure")
    ops.linear(w, x, y, n_tok, ws)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print(name, n_tok, n_out, k, algorithmic_bytes(n_tok, n_out, k))


if __name__ == "__main__":
    if sys.argv[1] == "shapes":
        print(" ".join(SHAPES))
    else:
        run(sys.argv[2])
