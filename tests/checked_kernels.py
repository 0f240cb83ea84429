"""TEST-ONLY debugging backend: every call runs the real C-ABI kernel and the
torch reference (tests/cpu_kernels.py) on cloned inputs, and reports the
first op whose outputs disagree. Use as ``Engine(..., kernels=checked_kernels)``."""

from __future__ import annotations

import torch

import cpu_kernels as ref
from paper_2311_11514_b200 import ops

LOG = []
TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def _rel(a, b):
    a, b = a.float(), b.float()
    den = b.abs().max().clamp_min(1e-20)
    return float((a - b).abs().max() / den)


def _wrap(name, outs):
    real = getattr(ops, name)
    rfn = getattr(ref, name)

    def fn(*args, **kw):
        cl = [a.clone() if isinstance(a, torch.Tensor) else a for a in args]
        real(*args, **kw)
        rfn(*cl, **kw)
        torch.cuda.synchronize()
        for i in outs:
            a, b = args[i], cl[i]
            if a is None:
                continue
            e = _rel(a, b)
            if e > TOL.get(a.dtype, 0) or torch.isnan(a.float()).any():
                shapes = [tuple(x.shape) if isinstance(x, torch.Tensor) else x for x in args]
                LOG.append((name, i, e, shapes))
                print(f"MISMATCH {name} out#{i} rel={e:.3e} shapes={shapes}")
    return fn


embed = _wrap("embed", [2])
rmsnorm = _wrap("rmsnorm", [2])
residual_add_rmsnorm = _wrap("residual_add_rmsnorm", [0, 3])
linear = _wrap("linear", [2])
swiglu = _wrap("swiglu", [1])
rope_kv_append = _wrap("rope_kv_append", [1, 2, 3])
attn_decode = _wrap("attn_decode", [5])
attn_prefill = _wrap("attn_prefill", [5])
advance = _wrap("advance", [0])
argmax_partial = _wrap("argmax_partial", [1])
argmax_finalize = ops.argmax_finalize
linear_workspace = ops.linear_workspace
attn_decode_workspace = ops.attn_decode_workspace
launch_count = ops.launch_count
