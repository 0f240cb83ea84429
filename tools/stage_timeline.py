"""Per-CTA timeline of one TP stage's decode step on real ranks (torchrun):
rank 0 records its stream-K GEMMs and decode attention (hx_debug_trace) in the
engine's own decode graph, so the NVLink all-reduces sit between the GEMMs as
in the bench. Prints, per GEMM role, the wait after the previous traced kernel,
the run after the wait and the tail, plus the QKV -> attention -> O phases.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/stage_timeline.py --tp 4 --layers 20
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import torch.distributed as dist

from paper_2311_11514_b200 import ops
from paper_2311_11514_b200.config import preset
from paper_2311_11514_b200.engine import Engine
from paper_2311_11514_b200.plan import simple_plan

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama2-70b")
ap.add_argument("--tp", type=int, default=4)
ap.add_argument("--layers", type=int, default=20)
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--s-in", type=int, default=1024)
a = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if a.tp > 1:
    dist.init_process_group("nccl", device_id=dev)
rank = dist.get_rank() if a.tp > 1 else 0
cfg = preset(a.model, num_layers=a.layers)
eng = Engine(simple_plan([a.tp], [a.layers]), cfg, dtype="bf16", batch=a.batch, max_prompt=a.s_in, max_out=8,
             comm="dist" if a.tp > 1 else "local", device=dev, weights="device")
prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(a.batch, a.s_in), dtype=np.int32)
eng.generate(prompt, 8)
lib = ops.load()
cap = 400 * 1024
buf = torch.zeros(cap * 8, dtype=torch.int64, device=dev)
if rank == 0:
    lib.hx_debug_trace(buf.data_ptr(), cap)
eng._graph_cache.clear()           # recapture with the trace armed (rank 0)
eng.generate(prompt, 8)
used = lib.hx_debug_trace(None, 0) if rank == 0 else 0
torch.cuda.synchronize()
if rank == 0:
    tr = buf.view(-1, 8)[:used].cpu().numpy().astype(np.int64)
    kind_of = np.where((tr[:, 3] >> 40) & 1, 1, np.where((tr[:, 3] >> 41) & 1, 2, 0))  # 0 GEMM, 1 attn, 2 AR
    launches, i = [], 0
    while i < used:
        if kind_of[i]:
            j = i
            while j < used and kind_of[j] == kind_of[i]:
                j += 1
            launches.append(("attn" if kind_of[i] == 1 else "ar", tr[i:j]))
            i = j
        else:
            launches.append(("gemm", tr[i:i + 148]))
            i += 148
    has_ar = any(k == "ar" for k, _ in launches)
    # anchor on the attention launches: [prev AR,] QKV, attention, O, [AR,] gate/up, down[, AR]
    names = ["qkv", "attn", "o", "ar1", "gu", "down", "ar2"] if has_ar else ["qkv", "attn", "o", "gu", "down"]
    lead = 2 if has_ar else 2
    stats = {n: [] for n in names}
    layer = []
    att_idx = [k for k, (kind, _) in enumerate(launches) if kind == "attn"]
    for k in att_idx:
        if k < lead or k - 1 + len(names) > len(launches):
            continue
        seq = launches[k - lead:k - 1 + len(names)]   # the previous layer's last launch, then this layer's
        st = [r[:, 0].min() for _, r in seq]
        if any(st[j + 1] < st[j] or st[j + 1] - st[j] > 1_000_000 for j in range(len(st) - 1)):
            continue                  # slots of an eager launch (stale) or a step boundary
        if [kd for kd, _ in seq[1:]] != [("attn" if n == "attn" else "ar" if n.startswith("ar") else "gemm")
                                         for n in names]:
            continue
        for j, nm in enumerate(names):
            kind, r = seq[j + 1]
            prev_end = seq[j][1][:, 2].max()
            us = lambda v: (v - prev_end) / 1e3
            if kind == "gemm":
                stats[nm].append((us(r[:, 1].min()), (r[:, 2].max() - r[:, 1].min()) / 1e3,
                                  (r[:, 2].max() - np.median(r[:, 2])) / 1e3))
            elif kind == "attn":
                stats[nm].append((us(np.median(r[:, 4])), us(r[:, 2][r[:, 2] > 0].max()), 0.0))
            else:   # all-reduce: wait done, partial read, pushed, peers arrived, end (max over CTAs)
                stats[nm].append((us(r[:, 1].max()), us(r[:, 4].max()), us(r[:, 5].max()), us(np.median(r[:, 6])),
                                  us(r[:, 6].max()), us(r[:, 2].max())))
        layer.append((seq[-1][1][:, 2].max() - seq[0][1][:, 2].max()) / 1e3)
    n = len(stats["qkv"])
    med = lambda v, c: float(np.median(v[:, c]))
    print(f"{a.model} TP={a.tp} x {a.layers} layers, b={a.batch}, ctx {a.s_in}: rank 0, {n} layers of one decode step (us)")
    for nm in names:
        v = np.array(stats[nm])
        if nm == "attn":
            print(f"  attention: q ready {med(v, 0):6.2f}  end {med(v, 1):6.2f} after the QKV GEMM's end")
        elif nm.startswith("ar"):
            print(f"  {nm:5s}: after the previous GEMM's end: wait done {med(v, 0):6.2f}  partial read {med(v, 1):6.2f}  "
                  f"pushed {med(v, 2):6.2f}  peers arrived med/max {med(v, 3):6.2f}/{med(v, 4):6.2f}  end {med(v, 5):6.2f}")
        else:
            print(f"  {nm:5s}: wait after previous traced kernel {med(v, 0):6.2f}  run after wait "
                  f"{med(v, 1):6.2f}  tail {med(v, 2):5.2f}")
    print(f"  per layer: median {np.median(layer):.1f} us  (medians over layers)")
if a.tp > 1:
    dist.barrier()
os._exit(0)
