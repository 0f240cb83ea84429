"""One tcgen05 prefill-attention launch (7B b=8 s=512, or 70B TP=1 micro-batch) in NVTX range "pfattn" (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2311_11514_b200 import ops

b, s, hq, hkv = (2, 1024, 64, 8) if "70b" in sys.argv else (8, 512, 32, 32)
hd, page = 128, 64
maxb = s // page
nb = b * maxb
ops.load()
kc = torch.randn(nb, hkv, page, hd, device="cuda").bfloat16()
bt = torch.randperm(nb, device="cuda", dtype=torch.int32).view(b, maxb).contiguous()
q = torch.randn(b * s, hq * hd, device="cuda").bfloat16()
o = torch.empty_like(q)
vt = torch.randn(b * hkv * hd * s, device="cuda").bfloat16()
for _ in range(3):
    ops.attn_prefill_tc(q, kc, vt, bt, o, b, s, hq, hkv, hd)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("pfattn")
ops.attn_prefill_tc(q, kc, vt, bt, o, b, s, hq, hkv, hd)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
