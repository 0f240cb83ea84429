"""Per-CTA timeline of the decode attention inside a real decode step
(hx_debug_trace records the stream-K GEMMs and the TMA decode attention),
replayed in a CUDA graph: where the QKV GEMM -> attention -> O GEMM
transition spends its time.

    python tools/attn_timeline.py [llama2-7b | llama2-70b --tp=4]

All times in us relative to the QKV GEMM's last CTA exit (negative = before it).
"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2311_11514_b200 import ops
from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.plan import simple_plan

model = next((a for a in sys.argv[1:] if not a.startswith("-")), "llama2-7b")
cfg = preset(model)
b, s_in = 8, 512
tp = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--tp=")), "1"))
if tp > 1:
    cfg = replace(cfg, head_dim_override=cfg.head_dim, num_heads=cfg.num_heads // tp, num_kv_heads=cfg.num_kv_heads // tp,
                  intermediate=cfg.intermediate // tp, vocab=cfg.vocab // tp)
if model == "llama2-70b":
    b, s_in = 32, 1024
    cfg = replace(cfg, num_layers=20)
eng = Engine(simple_plan([1], [cfg.num_layers]), cfg, dtype="bf16", batch=b, max_prompt=s_in, max_out=4,
             device="cuda:0", weights="device", use_graphs=False)
prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(b, s_in), dtype=np.int32)
eng.generate(prompt, 2)
lib = ops.load()
cap = 400 * 1024
buf = torch.zeros(cap * 8, dtype=torch.int64, device="cuda")
eng._reset(b, s_in, 4)
for ex in eng.execs:  # decode at context s_in (the prompt's pages), not an empty cache
    ex.kv.seq_lens.fill_(s_in)
lib.hx_debug_trace(buf.data_ptr(), cap)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    eng._decode_compute(eng.drivers[0], b)
used = lib.hx_debug_trace(None, 0)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
tr = buf.view(-1, 8)[:used].cpu().numpy().astype(np.int64)
is_attn = (tr[:, 3] >> 40) & 1
# split the record stream into launches: runs of attention records, GEMMs of sk_grid CTAs
launches, i = [], 0
G = 148
while i < used:
    if is_attn[i]:
        j = i
        while j < used and is_attn[j]:
            j += 1
        launches.append(("attn", tr[i:j]))
        i = j
    else:
        launches.append(("gemm", tr[i:i + G]))
        i += G
rows = []
for k, (kind, r) in enumerate(launches):
    if kind != "attn" or k == 0 or k + 1 >= len(launches):
        continue
    q_end = launches[k - 1][1][:, 2].max()
    o = launches[k + 1][1]
    us = lambda v: (v - q_end) / 1e3
    ends = r[:, 2][r[:, 2] > 0]
    comb = r[:, 6][r[:, 6] > 0]
    rows.append([us(r[:, 0].min()), us(r[:, 0].max()), us(r[:, 1].min()), us(r[:, 1].max()),
                 us(np.median(r[:, 4])), us(r[:, 4].max()), us(np.median(r[:, 5])), us(r[:, 5].max()),
                 us(comb.max()) if len(comb) else np.nan, us(ends.max()), us(o[:, 1].min()),
                 us(o[:, 2].max()), (r[:, 7] & 0xffff).max(), len(r)])
a = np.array(rows)
cols = ["attn start min", "attn start max", "wait done min", "wait done max", "q ready med", "q ready max",
        "loop done med", "loop done max", "combine sync max", "attn end max", "O wait release", "O end"]
print(f"{model} tp={tp} b={b}: {len(rows)} layers, attention CTAs {int(a[0, -1])}, max blocks per CTA {int(a[0, -2])}")
for c, name in enumerate(cols):
    print(f"  {name:18s} {a[:, c].mean():8.2f} us  (min {a[:, c].min():7.2f}, max {a[:, c].max():7.2f})")
# per-CTA loop time vs blocks
r = launches[[k for k, (kd, _) in enumerate(launches) if kd == "attn"][len(rows) // 2]][1]
nb = r[:, 7] & 0xffff
for v in sorted(set(nb.tolist())):
    sel = nb == v
    print(f"  CTAs with {v} blocks: {sel.sum():4d}, loop (q ready -> loop done) med "
          f"{np.median((r[sel, 5] - r[sel, 4]) / 1e3):.2f} us, wait->q ready med {np.median((r[sel, 4] - r[sel, 1]) / 1e3):.2f} us")
