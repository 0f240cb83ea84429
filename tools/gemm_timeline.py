"""Per-CTA timeline of the decode GEMMs (hx_debug_trace), replayed in a CUDA graph.

    python tools/gemm_timeline.py [llama2-7b] [--full-step]

Prints, per GEMM launch: span (first CTA start -> last CTA end), the spread
of CTA start times, how long after the previous GEMM's last CTA exit this
GEMM's CTAs passed griddepcontrol.wait, and the end-time spread (tail).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2311_11514_b200 import ops
from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.plan import simple_plan

model = next((a for a in sys.argv[1:] if not a.startswith("-")), "llama2-7b")
full = "--full-step" in sys.argv
cfg = preset(model)
b, s_in = 8, 512
# --tp N: one TP rank of a stage, as a single-GPU model whose layers have exactly
# that rank's shard shapes (heads, kv heads, intermediate and vocab divided by N)
tp = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--tp=")), "1"))
if tp > 1:
    from dataclasses import replace
    cfg = replace(cfg, head_dim_override=cfg.head_dim, num_heads=cfg.num_heads // tp, num_kv_heads=cfg.num_kv_heads // tp,
                  intermediate=cfg.intermediate // tp, vocab=cfg.vocab // tp)
if model == "llama2-70b":
    b, s_in = 32, 1024
    cfg = __import__("dataclasses").replace(cfg, num_layers=int(next(
        (a.split("=")[1] for a in sys.argv if a.startswith("--layers=")), "20")))
eng = Engine(simple_plan([1], [cfg.num_layers]), cfg, dtype="bf16", batch=b, max_prompt=s_in, max_out=4,
             device="cuda:0", weights="device", use_graphs=False)
prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(b, s_in), dtype=np.int32)
eng.generate(prompt, 2)
e = eng.execs[0]
lib = ops.load()
cap = 200 * 148
buf = torch.zeros(cap * 8, dtype=torch.int64, device="cuda")
seq = []
for lw in e.w["layers"]:
    seq += [(lw["wqkv"], e.h, e.qkv), (lw["wo"], e.attn, e.proj), (lw["wgu"], e.h, e.gu), (lw["wdown"], e.a, e.proj)]
seq.append((e.w["lm_head"], e.hl, e.logits))
lib.hx_debug_trace(buf.data_ptr(), cap)
if full:
    eng._reset(b, s_in, 4)
    for ex in eng.execs:  # decode at context s_in (the prompt's pages), not an empty cache
        ex.kv.seq_lens.fill_(s_in)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    if full:
        eng._decode_compute(eng.drivers[0], b)
    else:
        for wt, xin, y in seq:
            ops.linear(wt, xin, y, b, e.lin_ws)
used = lib.hx_debug_trace(None, 0)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
tr = buf.view(-1, 8)[:used].cpu().numpy().astype(np.int64)
tr = tr[((tr[:, 3] >> 40) & 1) == 0]   # drop the decode attention's records (same trace)
used = len(tr)
G = 148
n = used // G
names = ["qkv", "o", "gu", "down"]
t0 = tr[:, 0].min()
prev_end = None
rows = []
for i in range(n):
    r = tr[i * G:(i + 1) * G]
    st, wd, en = r[:, 0] - t0, r[:, 1] - t0, r[:, 2] - t0
    gap = (wd.min() - prev_end) if prev_end is not None else 0
    rows.append((i, names[i % 4] if i < n - 1 else "lm_head", (en.max() - st.min()) / 1e3,
                 (st.max() - st.min()) / 1e3, gap / 1e3, (en.max() - np.median(en)) / 1e3,
                 (en.max() - wd.max()) / 1e3))
    prev_end = en.max()
print(f"{'#':>4} {'gemm':8} {'span us':>8} {'start spread':>12} {'wait-after-prev':>15} {'tail(max-med end)':>17} {'run after wait':>14}")
for row in rows[:12] + rows[-2:]:
    print(f"{row[0]:4d} {row[1]:8s} {row[2]:8.2f} {row[3]:12.2f} {row[4]:15.2f} {row[5]:17.2f} {row[6]:14.2f}")
arr = np.array([r[2:] for r in rows[:-1]])
for k, name in enumerate(names):
    sel = arr[k::4]
    print(f"mean {name:6s}: span {sel[:, 0].mean():6.2f}  start-spread {sel[:, 1].mean():6.2f}  "
          f"wait-after-prev {sel[:, 2].mean():6.2f}  tail {sel[:, 3].mean():6.2f}  run-after-wait {sel[:, 4].mean():6.2f}")
total = (tr[:, 2].max() - tr[:, 0].min()) / 1e3
print(f"total wall of the traced GEMM sequence: {total:.1f} us over {n} launches")
# launch lead: previous GEMM's last CTA end - this GEMM's first CTA start (> 0: resident before it ended)
lead = [(tr[(i - 1) * G:i * G, 2].max() - tr[i * G:(i + 1) * G, 0].min()) / 1e3 for i in range(1, n)]
for k, name in enumerate(names):
    sel = lead[(k - 1) % 4::4]
    print(f"launch lead {name:6s}: mean {np.mean(sel):6.2f} us  min {np.min(sel):6.2f}  max {np.max(sel):6.2f}")

if "--detail" in sys.argv:
    for idx in (5, 6, 7):
        r = tr[idx * G:(idx + 1) * G].copy()
        wd, en, sm = r[:, 1], r[:, 2], r[:, 3]
        base = wd.min()
        run = (en - base) / 1e3
        order = np.argsort(run)
        print(f"launch {idx} ({names[idx % 4]}): end-after-first-wait (us) min {run.min():.2f} med {np.median(run):.2f} max {run.max():.2f}")
        print("  slowest CTAs (cta, smid, wait_off, end_off):",
              [(int(c), int(sm[c]), round((wd[c] - base) / 1e3, 2), round(run[c], 2)) for c in order[-8:]])
        print("  fastest CTAs:", [(int(c), int(sm[c]), round((wd[c] - base) / 1e3, 2), round(run[c], 2)) for c in order[:5]])
        # correlation with CTA index parity / SM die halves
        def ev(cc):
            rr = r[cc]
            f = lambda v: round((v - base) / 1e3, 2) if v else None
            return dict(cta=int(cc), acc0=f(rr[4]), acc_last=f(rr[6]), fenced=f(rr[5]), ticket=f(rr[7]), end=f(rr[2]))
        print("  slow:", [ev(cc) for cc in order[-4:]])
        print("  fast:", [ev(cc) for cc in order[:3]])
        print("  mean end by smid<74 vs >=74:", round(run[sm < 74].mean(), 2), round(run[sm >= 74].mean(), 2),
              " by cta index quartile:", [round(run[q * 37:(q + 1) * 37].mean(), 2) for q in range(4)])
