"""Profiling driver: one Llama prefill (b=8, s=512) inside an NVTX range "prefill":
NVTX ranges so ncu can select one decode step:
  ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum ... python tools/profile_decode.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.plan import simple_plan

model = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
b, s_in = 8, 512
cfg = preset(model)
eng = Engine(simple_plan([1], [cfg.num_layers]), cfg, dtype="bf16", batch=b, max_prompt=s_in, max_out=4,
             device="cuda:0", weights="device", use_graphs=False)
prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(b, s_in), dtype=np.int32)
eng.generate(prompt, 2)
torch.cuda.synchronize()
# one more request: prefill outside the range, decode steps inside
eng._reset(b, s_in, 4)
for e in eng.execs:
    e.prompt[:b * s_in].copy_(torch.from_numpy(prompt.reshape(-1)))
torch.cuda.nvtx.range_push("prefill")
eng._prefill(b, s_in)
torch.cuda.nvtx.range_pop()
for t in range(0):
    torch.cuda.nvtx.range_push("decode")
    eng._decode_step(b, None)
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("profile_decode done")
