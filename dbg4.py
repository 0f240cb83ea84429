import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.plan import simple_plan
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.weights import synthetic_prompts, init_host_weights
from oracle import llama_oracle as O
cfg = preset("llama2-7b", num_layers=1)
b,s=8,64
prompt=synthetic_prompts(cfg,b,s,1)
w=O.bf16_weights(init_host_weights(cfg,0))
eng=Engine(simple_plan([1],[1]), cfg, dtype='bf16', batch=b, max_prompt=s, max_out=2, device='cuda:0', use_graphs=False)
e=eng.execs[0]
eng._reset(b,s,2)
e.prompt[:b*s].copy_(torch.from_numpy(prompt.reshape(-1)))
eng._prefill(b,s)
torch.cuda.synchronize()
r=O.bf16_round; lw=w["layers"][0]
x0=w["embed"][prompt].astype(np.float32).reshape(b*s,-1)
h=r(O.rmsnorm(x0,lw["ln_attn"],cfg.rms_eps))
qkv=np.concatenate([r(O.lin(h,lw["q"])),r(O.lin(h,lw["k"])),r(O.lin(h,lw["v"]))],-1)
def cmp(name, a, ref):
    a=a.float().cpu().numpy().reshape(ref.shape)
    d=np.abs(a-ref); print(f"{name:6s} maxrel {d.max()/np.abs(ref).max():.3e} rms-rel {np.sqrt((d**2).mean()/(ref**2).mean()):.3e}")
cmp('qkv', e.qkv[:b*s], qkv)
hd=128; H=4096
q=qkv[:,:H].reshape(b,s,32,hd).transpose(0,2,1,3); k=qkv[:,H:2*H].reshape(b,s,32,hd).transpose(0,2,1,3); v=qkv[:,2*H:].reshape(b,s,32,hd).transpose(0,2,1,3)
cos,sin=O.rope_tables(hd,cfg.rope_theta,np.arange(s))
q=r(O.apply_rope(q,cos,sin)); k=r(O.apply_rope(k,cos,sin))
cmp('q', e.q[:b*s], q.transpose(0,2,1,3).reshape(b*s,H))
o=r(O.attention(q,k,v,0)).transpose(0,2,1,3).reshape(b*s,H)
cmp('attn', e.attn[:b*s], o)
x1=(x0+O.lin(o,lw["o"])).astype(np.float32)
h2=r(O.rmsnorm(x1,lw["ln_mlp"],cfg.rms_eps))
g=r(O.lin(h2,lw["gate"])); u=r(O.lin(h2,lw["up"]))
cmp('gu', e.gu[:b*s], np.concatenate([g,u],-1))
a=r(O.silu(g)*u)
cmp('act', e.a[:b*s], a)
x2=(x1+O.lin(a,lw["down"])).astype(np.float32)
cmp('x', e.x[:b*s], x2)
# same checks fed with the engine's own inputs (isolates each kernel)
def t2n(t): return t.float().cpu().numpy()
cmp('attn|eng-in', e.attn[:b*s], r(O.attention(t2n(e.q[:b*s]).reshape(b,s,32,hd).transpose(0,2,1,3), k, v, 0)).transpose(0,2,1,3).reshape(b*s,H))
ae=t2n(e.attn[:b*s])
x1e=(x0+O.lin(ae,lw["o"])).astype(np.float32)
h2e=r(O.rmsnorm(x1e,lw["ln_mlp"],cfg.rms_eps))
cmp('gu|eng-attn', e.gu[:b*s], np.concatenate([r(O.lin(h2e,lw["gate"])),r(O.lin(h2e,lw["up"]))],-1))
print('x1 scale', np.abs(x1).max(), np.sqrt((x1**2).mean()), 'x0', np.sqrt((x0**2).mean()))
print('h2 rel diff from attn diffs', np.sqrt(((h2e-h2)**2).mean()/(h2**2).mean()))
d=np.abs(t2n(e.attn[:b*s])-o).reshape(b,s,32,hd)
print('attn err by token pos', [float(d[:,i].max()) for i in (0,1,2,5,10,30,63)])
print('attn err by head', [float(d[:,:,hh].max()) for hh in range(0,32,4)])
