import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
import checked_kernels
from paper_2311_11514_b200.config import LlamaConfig, preset
from paper_2311_11514_b200.plan import simple_plan
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.weights import synthetic_prompts
cfg = preset("llama2-7b", num_layers=2)
b,s,so=8,64,3
prompt=synthetic_prompts(cfg,b,s,1)
eng=Engine(simple_plan([1],[2]), cfg, dtype='bf16', batch=b, max_prompt=s, max_out=so, device='cuda:0', kernels=checked_kernels)
r=eng.generate(prompt, so, return_logits=True)
print("mismatches:", len(checked_kernels.LOG))
for l in checked_kernels.LOG[:20]: print(l)
