import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, collections
import checked_kernels
checked_kernels.TOL = {torch.float32: 0.0, torch.bfloat16: 0.0}
from paper_2311_11514_b200.config import LlamaConfig, preset
from paper_2311_11514_b200.plan import simple_plan
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.weights import synthetic_prompts
import builtins
_print = builtins.print
builtins.print = lambda *a, **k: None
cfg = preset("llama2-7b", num_layers=2)
b,s,so=8,64,3
prompt=synthetic_prompts(cfg,b,s,1)
eng=Engine(simple_plan([1],[2]), cfg, dtype='bf16', batch=b, max_prompt=s, max_out=so, device='cuda:0', kernels=checked_kernels, weights='host')
r=eng.generate(prompt, so, return_logits=True)
builtins.print = _print
agg=collections.defaultdict(list)
for name,i,e,shapes in checked_kernels.LOG:
    agg[(name,i,str(shapes[:3]))].append(e)
for k,v in agg.items(): print(k, len(v), max(v))
