import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
from paper_2311_11514_b200.config import LlamaConfig, preset
from paper_2311_11514_b200.plan import simple_plan
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.weights import synthetic_prompts, init_host_weights
from oracle.llama_oracle import Oracle, bf16_weights
for cfg,tps,layers,b,s,so,page in [(preset("llama2-7b", num_layers=2),[1],[2],8,64,6,64),(LlamaConfig("gqa-mini", 2, 2048, 16, 2, 5632, 32000),[2,1],[1,1],4,80,6,32)]:
    w=init_host_weights(cfg,0); prompt=synthetic_prompts(cfg,b,s,1)
    ids_o, lg_o = Oracle(cfg, bf16_weights(w)).generate(prompt, so)
    eng=Engine(simple_plan(tps,layers), cfg, dtype='bf16', batch=b, max_prompt=s, max_out=so, device='cuda:0', page_size=page)
    r=eng.generate(prompt, so, forced=ids_o)
    scale=np.abs(lg_o).max(-1,keepdims=True)
    err=np.abs(r.logits-lg_o)/scale
    print('err per step', err.max(axis=(1,2)))
    srt=np.sort(lg_o,-1); margin=(srt[...,-1]-srt[...,-2])/scale[...,0]
    print('margin min per step', margin.min(axis=1))
    print('oracle ids', ids_o[:2]); print('engine ids', r.ids[:2])
    dis = np.argwhere(r.ids.T != ids_o.T)
    for t,bb in dis[:10]: print('disagree t',t,'b',bb,'margin',margin[t,bb],'err',err[t,bb].max(), 'eng top', np.argsort(-r.logits[t,bb])[:3], 'orc top', np.argsort(-lg_o[t,bb])[:3])
