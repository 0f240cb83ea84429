"""One decode-attention launch at a config shape inside NVTX range "attn" (for ncu).

    ncu --set full --nvtx --nvtx-include attn/ -k regex:attn_decode_tma python tools/attn_profile.py [shape]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2311_11514_b200 import ops
from tools.attn_bench import SHAPES

name = next((k for k in SHAPES if len(sys.argv) > 1 and sys.argv[1] in k), "70b tp4 b32 ctx1151")
b, hq, hkv, ctx = SHAPES[name]
hd, page = 128, 64
maxb = (ctx + 1 + page - 1) // page + 1
nb = b * maxb
ops.load()
kc = torch.randn(nb, hkv, page, hd, device="cuda").bfloat16()
vc = torch.randn(nb, hkv, page, hd, device="cuda").bfloat16()
bt = torch.randperm(nb, device="cuda", dtype=torch.int32).view(b, maxb).contiguous()
sl = torch.full((b,), ctx - 1, dtype=torch.int32, device="cuda")
qkv = torch.randn(b, (hq + 2 * hkv) * hd, device="cuda").bfloat16()
o = torch.empty(b, hq * hd, device="cuda").bfloat16()
ws = torch.zeros(max(ops.attn_decode_workspace(b, hq, hkv, hd, maxb * page), 256) // 4 + 64, dtype=torch.int32,
                 device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ops.attn_decode_rope_append(qkv, kc, vc, bt, sl, o, b, hq, hkv, hd, maxb * page, 1e4, ws)
flush.zero_()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("attn")
ops.attn_decode_rope_append(qkv, kc, vc, bt, sl, o, b, hq, hkv, hd, maxb * page, 1e4, ws)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print(name, "done")
