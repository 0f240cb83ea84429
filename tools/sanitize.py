"""Small invocations of every hx kernel family, one process, everything on one
stream -- a quick all-kernels check, and the input for compute-sanitizer
(memcheck / racecheck / synccheck) where it is available (it is closed on the
gpurun pool this repo was measured on):

    python tools/sanitize.py
    compute-sanitizer --tool memcheck python tools/sanitize.py

The multi-rank spin protocols (push all-reduce, concurrent hand-offs) need
their partner kernels running concurrently, which the sanitizer's serialised
launches cannot give, so they run here in their sequential forms only: the
hand-off push then pull on one stream, and the flow-controlled (credit)
stream of hand-offs, push before pull each time.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2311_11514_b200 import ops

DEV = "cuda"
g = torch.Generator(device=DEV).manual_seed(0)
bf = torch.bfloat16


def ws_for(n_tok, n_out, k):
    return torch.zeros(ops.linear_workspace(bf, n_tok, n_out, k) // 4 + 64, dtype=torch.int32, device=DEV)


def gemms():
    for n_tok, n_out, k in ((8, 1024, 512), (32, 640, 1024), (300, 768, 256)):
        w = ops.PackedWeight((torch.randn(n_out, k, device=DEV, generator=g) * 0.02).to(bf))
        x = torch.randn(n_tok, k, device=DEV, generator=g).to(bf)
        y = torch.empty(n_tok, n_out, device=DEV)
        ws = ws_for(n_tok, n_out, k)
        ops.linear(w, x, y, n_tok, ws)
        if n_tok <= 64:   # deferred split-K + its consumers
            ops.linear(w, x, y, n_tok, ws, defer_reduce=True)
            xr = torch.randn(n_tok, n_out, device=DEV)
            gain = torch.ones(n_out, device=DEV)
            ops.splitk_residual_rmsnorm(xr, y, ws, n_tok, k, gain, torch.empty(n_tok, n_out, device=DEV, dtype=bf),
                                        1e-5)
    print("gemms ok", flush=True)


def attention():
    b, hq, hkv, hd, page, ctx = 4, 8, 2, 128, 64, 130
    mb = (ctx + 1 + page - 1) // page
    kc = torch.zeros(b * mb, hkv, page, hd, device=DEV, dtype=bf)
    vc = torch.zeros_like(kc)
    bt = torch.randperm(b * mb, generator=g, device=DEV).to(torch.int32).view(b, mb).contiguous()
    n = (hq + 2 * hkv) * hd
    seq = torch.zeros(b, dtype=torch.int32, device=DEV)
    hist = torch.randn(b * ctx, n, device=DEV, generator=g).to(bf)
    ops.rope_kv_append(hist, torch.empty(b * ctx, hq * hd, device=DEV, dtype=bf), kc, vc, bt, seq, b * ctx, ctx,
                       hq, hkv, hd, 10000.0)
    seq.fill_(ctx)
    aws = torch.zeros(ops.attn_decode_workspace(b, hq, hkv, hd, ctx + 1) // 4 + 64, dtype=torch.int32, device=DEV)
    new = torch.randn(b, n, device=DEV, generator=g).to(bf)
    o = torch.empty(b, hq * hd, device=DEV, dtype=bf)
    ops.attn_decode_rope_append(new, kc, vc, bt, seq, o, b, hq, hkv, hd, ctx + 1, 10000.0, aws)
    w = ops.PackedWeight((torch.randn(n, 512, device=DEV, generator=g) * 0.02).to(bf))
    x = torch.randn(b, 512, device=DEV, generator=g).to(bf)
    lws = ws_for(b, n, 512)
    q32 = torch.empty(b, n, device=DEV)
    ops.linear(w, x, q32, b, lws, defer_reduce=True)
    ops.attn_decode_rope_append_sk(q32, lws, 512, kc, vc, bt, seq, o, b, hq, hkv, hd, ctx + 1, 10000.0, aws)
    # prefill attention (tcgen05, s = 128) on a fresh cache
    s = 128
    seq.zero_()
    qkv = torch.randn(b * s, n, device=DEV, generator=g).to(bf)
    q = torch.empty(b * s, hq * hd, device=DEV, dtype=bf)
    ops.rope_kv_append(qkv, q, kc, vc, bt, seq, b * s, s, hq, hkv, hd, 10000.0)
    vt = torch.empty(b * s * hkv * hd, device=DEV, dtype=bf)
    ops.prefill_vt(qkv, vt, b, s, hq, hkv, hd)
    ops.attn_prefill_tc(q, kc, vt, bt, torch.empty_like(q), b, s, hq, hkv, hd)
    ops.attn_prefill(q, kc, vc, bt, seq, torch.empty_like(q), b, s, hq, hkv, hd)
    print("attention ok", flush=True)


def handoffs():
    words = 4096
    link, stream = ops.P2PLink.local(0, 1, words), ops.P2PLink.local(0, 1, words)   # one protocol per link
    for k in range(5):
        src = torch.randn(words - 4 * (k % 2), device=DEV, generator=g)
        dst = torch.empty_like(src)
        link.push(src)
        link.pull(dst)
        stream.push_credit(src)
        stream.pull_credit(dst)
    link.close()
    stream.close()
    print("handoffs ok", flush=True)


def elementwise():
    n_tok, H, V = 4, 512, 1000
    x = torch.randn(n_tok, H, device=DEV, generator=g)
    gain = torch.ones(H, device=DEV)
    out = torch.empty(n_tok, H, device=DEV, dtype=bf)
    ops.rmsnorm(x, gain, out, n_tok, 1e-5)
    ops.residual_add_rmsnorm(x, torch.randn(n_tok, H, device=DEV, generator=g), gain, out, n_tok, 1e-5)
    gu = torch.randn(n_tok, 2 * H, device=DEV, generator=g).to(bf)
    ops.swiglu(gu, torch.empty(n_tok, H, device=DEV, dtype=bf), n_tok)
    table = torch.randn(V, H, device=DEV, generator=g).to(bf)
    ids = torch.randint(0, V, (n_tok,), device=DEV, dtype=torch.int32, generator=g)
    ops.embed(ids, table, x, n_tok)
    logits = torch.randn(n_tok, V, device=DEV, generator=g)
    keys = torch.empty(n_tok, dtype=torch.int64, device=DEV)
    ops.argmax_partial(logits, keys, n_tok, V, 0)
    hist = torch.zeros(n_tok, 4, dtype=torch.int32, device=DEV)
    ops.argmax_finalize(keys, ids, hist, torch.zeros(1, dtype=torch.int32, device=DEV), n_tok)
    print("elementwise ok", flush=True)


if __name__ == "__main__":
    ops.load()
    gemms()
    attention()
    handoffs()
    elementwise()
    torch.cuda.synchronize()
    print("sanitize run complete", flush=True)
