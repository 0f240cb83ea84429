"""Kernel-level parity on the B200: every hx_* entry point against a plain
PyTorch fp32 reference of the same op (bf16 inputs upcast exactly)."""

import math

import numpy as np
import pytest
import torch

import cpu_kernels as ref
from paper_2311_11514_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"


def rel_err(a, b):
    a, b = a.float(), b.float()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.fixture(autouse=True, scope="module")
def _lib():
    ops.load()


# ------------------------------------------------------------------ linear
DECODE_SHAPES = [(8, 12288, 4096), (8, 4096, 4096), (8, 22016, 4096), (8, 4096, 11008), (8, 32000, 4096),
                 (32, 2560, 8192), (32, 8192, 2048), (2, 768, 256), (1, 4096, 4096), (16, 1000, 520),
                 (33, 384, 128), (64, 16000, 8192)]
PREFILL_SHAPES = [(4096, 12288, 4096), (4096, 4096, 11008), (300, 768, 256), (130, 1000, 520), (65, 32000, 256)]


@pytest.mark.parametrize("n_tok,n_out,k", DECODE_SHAPES + PREFILL_SHAPES)
@pytest.mark.parametrize("ydt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("packed", [False, True])
def test_linear_bf16(n_tok, n_out, k, ydt, packed):
    g = torch.Generator(device=DEV).manual_seed(n_tok * 7 + n_out + k)
    w = (torch.randn(n_out, k, device=DEV, generator=g) * 0.02).bfloat16()
    x = torch.randn(n_tok, k, device=DEV, generator=g).bfloat16()
    y = torch.full((n_tok, n_out), float("nan"), device=DEV, dtype=ydt)
    ws = torch.zeros(ops.linear_workspace(torch.bfloat16, n_tok, n_out, k) // 4 + 64, dtype=torch.int32, device=DEV)
    wl = ops.PackedWeight(w) if packed else w
    ops.linear(wl, x, y, n_tok, ws)
    torch.cuda.synchronize()
    want = x.float() @ w.float().T
    tol = 2e-5 * math.sqrt(k) if ydt == torch.float32 else 8e-3
    assert not torch.isnan(y).any()
    assert rel_err(y, want) < tol
    # ticket counters are re-armed: a second launch gives identical bits
    y2 = torch.empty_like(y)
    ops.linear(wl, x, y2, n_tok, ws)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)


def test_linear_shared_workspace_across_shapes():
    """The engine shares one split-K workspace across GEMMs of different tile
    counts; a small-tile GEMM must not clobber the big one's tickets."""
    shapes = [(8, 4096, 4096), (8, 12288, 4096), (8, 4096, 11008), (8, 22016, 4096), (8, 32000, 4096)]
    ws = torch.zeros(max(ops.linear_workspace(torch.bfloat16, *s) for s in shapes) // 4 + 64,
                     dtype=torch.int32, device=DEV)
    for _ in range(2):
        for n_tok, n_out, k in shapes:
            w = (torch.randn(n_out, k, device=DEV) * 0.02).bfloat16()
            x = torch.randn(64, k, device=DEV).bfloat16()   # buffer taller than n_tok
            y = torch.zeros(64, n_out, device=DEV)
            ops.linear(w, x, y, n_tok, ws)
            torch.cuda.synchronize()
            assert rel_err(y[:n_tok], x[:n_tok].float() @ w.float().T) < 1e-3
            assert not y[n_tok:].any()


def test_pack_weight_layout():
    w = torch.randn(300, 200, device=DEV).bfloat16()   # ragged in both dims -> zero padding
    pw = ops.PackedWeight(w)
    torch.cuda.synchronize()
    t = pw.data.view(3, 4, 128, 64)
    pad = torch.zeros(384, 256, device=DEV, dtype=torch.bfloat16)
    pad[:300, :200] = w
    want = pad.view(3, 128, 4, 64).permute(0, 2, 1, 3)
    assert torch.equal(t, want)


def test_pdl_off_gives_identical_bits():
    w = ops.PackedWeight((torch.randn(4096, 4096, device=DEV) * 0.02).bfloat16())
    x = torch.randn(8, 4096, device=DEV).bfloat16()
    ws = torch.zeros(ops.linear_workspace(torch.bfloat16, 8, 4096, 4096) // 4 + 64, dtype=torch.int32, device=DEV)
    y1, y2 = torch.empty(8, 4096, device=DEV), torch.empty(8, 4096, device=DEV)
    ops.linear(w, x, y1, 8, ws)
    ops.set_pdl(False)
    try:
        ops.linear(w, x, y2, 8, ws)
    finally:
        ops.set_pdl(True)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("n_tok,inter,k", [(8, 11008, 4096), (32, 7168, 8192), (3, 1408, 512), (32, 14336, 8192)])
def test_deferred_gate_up_swiglu_bit_identical(n_tok, inter, k):
    """linear(defer_reduce) into fp32 + splitk_swiglu == linear (bf16 gu) + swiglu, bitwise."""
    w = ops.PackedWeight((torch.randn(2 * inter, k, device=DEV) * 0.02).bfloat16())
    x = torch.randn(64, k, device=DEV).bfloat16()
    ws = torch.zeros(ops.linear_workspace(torch.bfloat16, n_tok, 2 * inter, k) // 4 + 64, dtype=torch.int32,
                     device=DEV)
    gu = torch.empty(64, 2 * inter, device=DEV, dtype=torch.bfloat16)
    a1 = torch.empty(64, inter, device=DEV, dtype=torch.bfloat16)
    ops.linear(w, x, gu, n_tok, ws)
    ops.swiglu(gu, a1, n_tok)
    y = torch.zeros(64, 2 * inter, device=DEV)
    a2 = torch.empty_like(a1)
    ops.linear(w, x, y, n_tok, ws, defer_reduce=True)
    ops.splitk_swiglu(y, ws, n_tok, k, a2)
    torch.cuda.synchronize()
    assert torch.equal(a1[:n_tok], a2[:n_tok])


@pytest.mark.parametrize("n_tok,H,k", [(8, 4096, 4096), (8, 4096, 11008), (32, 8192, 2048), (3, 2048, 5632),
                                       (1, 256, 768)])
def test_deferred_splitk_matches_in_kernel_reduction(n_tok, H, k):
    """linear(defer_reduce) + splitk_residual_rmsnorm == linear + residual_add_rmsnorm, bitwise."""
    w = ops.PackedWeight((torch.randn(H, k, device=DEV) * 0.02).bfloat16())
    a = torch.randn(64, k, device=DEV).bfloat16()
    gain = 1 + 0.1 * torch.randn(H, device=DEV)
    x0 = torch.randn(64, H, device=DEV)
    ws = torch.zeros(ops.linear_workspace(torch.bfloat16, n_tok, H, k) // 4 + 64, dtype=torch.int32, device=DEV)
    y = torch.zeros(64, H, device=DEV)
    x1, h1 = x0.clone(), torch.empty(64, H, device=DEV, dtype=torch.bfloat16)
    ops.linear(w, a, y, n_tok, ws)
    ops.residual_add_rmsnorm(x1, y, gain, h1, n_tok, 1e-5)
    x2, h2 = x0.clone(), torch.empty(64, H, device=DEV, dtype=torch.bfloat16)
    y2 = torch.zeros(64, H, device=DEV)
    ops.linear(w, a, y2, n_tok, ws, defer_reduce=True)
    ops.splitk_residual_rmsnorm(x2, y2, ws, n_tok, k, gain, h2, 1e-5)
    x3 = x0.clone()
    ops.linear(w, a, y2, n_tok, ws, defer_reduce=True)
    ops.splitk_residual_rmsnorm(x3, y2, ws, n_tok, k, None, None, 1e-5)   # add only
    torch.cuda.synchronize()
    assert torch.equal(x1[:n_tok], x2[:n_tok])  # the split-K sum is bitwise the in-kernel one
    # the norm's block reduction uses a different thread count: at most 1 bf16 ulp apart
    assert rel_err(h2[:n_tok], h1[:n_tok]) < 8e-3
    assert torch.equal(x3[:n_tok], x1[:n_tok])
    assert torch.equal(x2[n_tok:], x0[n_tok:])


def test_linear_bf16_accumulate_and_pitch():
    w = (torch.randn(512, 256, device=DEV) * 0.05).bfloat16()
    x = torch.randn(8, 256, device=DEV).bfloat16()
    y = torch.randn(8, 600, device=DEV)
    base = y.clone()
    ws = torch.zeros(ops.linear_workspace(torch.bfloat16, 8, 512, 256) // 4 + 64, dtype=torch.int32, device=DEV)
    ops.linear(w, x, y, 8, ws, accumulate=True)
    torch.cuda.synchronize()
    want = base.clone()
    want[:, :512] += x.float() @ w.float().T
    assert rel_err(y, want) < 1e-4
    assert torch.equal(y[:, 512:], base[:, 512:])


@pytest.mark.parametrize("n_tok,n_out,k", [(2, 768, 256), (128, 1536, 256), (130, 32000, 256), (1, 64, 768)])
def test_linear_f32(n_tok, n_out, k):
    w = torch.randn(n_out, k, device=DEV) * 0.02
    x = torch.randn(n_tok, k, device=DEV)
    y = torch.empty(n_tok, n_out, device=DEV)
    ops.linear(w, x, y, n_tok)
    torch.cuda.synchronize()
    want = (x.double() @ w.double().T).float()
    assert rel_err(y, want) < 1e-5


# ------------------------------------------------------------------ row ops
@pytest.mark.parametrize("H", [256, 4096, 5120, 8192])
@pytest.mark.parametrize("odt", [torch.float32, torch.bfloat16])
def test_norms(H, odt):
    x = torch.randn(9, H, device=DEV)
    d = torch.randn(9, H, device=DEV)
    gain = 1 + 0.1 * torch.randn(H, device=DEV)
    out = torch.empty(9, H, device=DEV, dtype=odt)
    want = torch.empty(9, H, device=DEV)
    ref.rmsnorm(x, gain, want, 9, 1e-5)
    ops.rmsnorm(x, gain, out, 9, 1e-5)
    torch.cuda.synchronize()
    assert rel_err(out, want) < (1e-6 if odt == torch.float32 else 8e-3)
    x2, x3 = x.clone(), x.clone()
    ops.residual_add_rmsnorm(x2, d, gain, out, 9, 1e-5)
    ref.residual_add_rmsnorm(x3, d, gain, want, 9, 1e-5)
    torch.cuda.synchronize()
    assert torch.allclose(x2, x3)
    assert rel_err(out, want) < (1e-6 if odt == torch.float32 else 8e-3)
    x4 = x.clone()
    ops.residual_add_rmsnorm(x4, d, None, None, 9, 1e-5)  # add only
    torch.cuda.synchronize()
    assert torch.allclose(x4, x + d)
    # strided rows (last prompt token of each sequence)
    xs = torch.randn(3, 5, H, device=DEV)
    out3 = torch.empty(3, H, device=DEV, dtype=odt)
    ops.rmsnorm(xs.view(-1)[4 * H:], gain, out3, 3, 1e-5, ldx=5 * H)
    want3 = torch.empty(3, H, device=DEV)
    ref.rmsnorm(xs[:, 4].contiguous(), gain, want3, 3, 1e-5)
    torch.cuda.synchronize()
    assert rel_err(out3, want3) < (1e-6 if odt == torch.float32 else 8e-3)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_embed_swiglu(dt):
    table = torch.randn(1000, 512, device=DEV).to(dt)
    ids = torch.tensor([0, 999, 5, 5, 123], dtype=torch.int32, device=DEV)
    x = torch.empty(5, 512, device=DEV)
    ops.embed(ids, table, x, 5)
    gu = torch.randn(7, 2 * 768, device=DEV).to(dt)
    a = torch.empty(7, 768, device=DEV, dtype=dt)
    ops.swiglu(gu, a, 7)
    torch.cuda.synchronize()
    assert torch.equal(x, table[ids.long()].float())
    want = torch.empty(7, 768, device=DEV)
    ref.swiglu(gu.float(), want, 7)
    assert rel_err(a, want) < (1e-6 if dt == torch.float32 else 8e-3)


def test_argmax_keys_and_ties():
    lg = torch.randn(4, 1000, device=DEV)
    lg[1, 10] = lg[1, 20] = 50.0           # tie -> first index
    lg[2] = -1.0
    lg[2, 999] = -0.5                      # all negative
    keys = torch.empty(4, dtype=torch.int64, device=DEV)
    ops.argmax_partial(lg, keys, 4, 1000, 0)
    ids = torch.empty(4, dtype=torch.int32, device=DEV)
    hist = torch.zeros(4, 3, dtype=torch.int32, device=DEV)
    step = torch.ones(1, dtype=torch.int32, device=DEV)
    ops.argmax_finalize(keys, ids, hist, step, 4)
    torch.cuda.synchronize()
    assert ids.tolist() == torch.argmax(lg, -1).tolist()
    assert hist[:, 1].tolist() == ids.tolist() and int(step) == 2
    # vocab-parallel: max over per-shard keys == global argmax
    shards = lg.chunk(4, dim=1)
    ks = []
    for r, s in enumerate(shards):
        k = torch.empty(4, dtype=torch.int64, device=DEV)
        ops.argmax_partial(s.contiguous(), k, 4, 250, r * 250)
        ks.append(k)
    kmax = torch.stack(ks).max(0).values
    ops.argmax_finalize(kmax, ids, None, None, 4)
    torch.cuda.synchronize()
    assert ids.tolist() == torch.argmax(lg, -1).tolist()


# ------------------------------------------------------------------ attention
def _paged_setup(dt, b, hq, hkv, hd, page, ctx_max, seed=0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    mb = math.ceil(ctx_max / page)
    nb = b * mb
    kc = torch.zeros(nb, hkv, page, hd, device=DEV, dtype=dt)
    vc = torch.zeros_like(kc)
    perm = torch.randperm(nb, generator=g, device=DEV).to(torch.int32)
    bt = perm.view(b, mb).contiguous()
    return kc, vc, bt, g


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("hq,hkv,hd,ctx", [(8, 8, 32, 70), (32, 32, 128, 600), (16, 2, 128, 1100),
                                            (64, 8, 128, 300), (4, 4, 64, 1), (8, 4, 128, 333),
                                            (16, 4, 64, 90), (16, 1, 128, 2), (32, 2, 128, 1279)])
@pytest.mark.parametrize("page", [16, 64])   # 64 with hd 128 takes the TMA-fed kernel
def test_rope_append_and_decode_attention(dt, hq, hkv, hd, ctx, page):
    b = 3
    kc, vc, bt, g = _paged_setup(dt, b, hq, hkv, hd, page, ctx + 1)
    kr, vr = kc.clone(), vc.clone()
    # fill ctx cached tokens with random K/V through the reference writer
    seq = torch.zeros(b, dtype=torch.int32, device=DEV)
    n = (hq + 2 * hkv) * hd
    hist = (torch.randn(b * ctx, n, device=DEV, generator=g)).to(dt)
    qo = torch.empty(b * ctx, hq * hd, device=DEV, dtype=dt)
    ops.rope_kv_append(hist, qo, kc, vc, bt, seq, b * ctx, ctx, hq, hkv, hd, 10000.0)
    ref.rope_kv_append(hist, qo.clone(), kr, vr, bt, seq, b * ctx, ctx, hq, hkv, hd, 10000.0)
    torch.cuda.synchronize()
    assert rel_err(kc, kr) < (1e-5 if dt == torch.float32 else 8e-3)
    assert torch.equal(vc, vr)
    seq.fill_(ctx)
    new = torch.randn(b, n, device=DEV, generator=g).to(dt)
    q = torch.empty(b, hq * hd, device=DEV, dtype=dt)
    qr = torch.empty_like(q)
    ops.rope_kv_append(new, q, kc, vc, bt, seq, b, 0, hq, hkv, hd, 10000.0)
    ref.rope_kv_append(new, qr, kr, vr, bt, seq, b, 0, hq, hkv, hd, 10000.0)
    o = torch.empty(b, hq * hd, device=DEV, dtype=dt)
    want = torch.empty(b, hq * hd, device=DEV)
    ws = torch.zeros(ops.attn_decode_workspace(b, hq, hkv, hd, ctx + 1) // 4 + 64, dtype=torch.int32, device=DEV)
    ops.attn_decode(q, kc, vc, bt, seq, o, b, hq, hkv, hd, ctx + 1, ws)
    ref.attn_decode(qr, kr, vr, bt, seq, want, b, hq, hkv, hd, ctx + 1)
    torch.cuda.synchronize()
    assert rel_err(q, qr) < (1e-5 if dt == torch.float32 else 8e-3)
    assert rel_err(o, want) < (2e-5 if dt == torch.float32 else 2e-2)
    o2 = torch.empty_like(o)
    ops.attn_decode(q, kc, vc, bt, seq, o2, b, hq, hkv, hd, ctx + 1, ws)
    torch.cuda.synchronize()
    assert torch.equal(o, o2)


@pytest.mark.parametrize("hq,hkv,ctx,b", [(32, 32, 600, 3), (32, 32, 575, 8), (16, 2, 1100, 3), (64, 8, 300, 2),
                                          (16, 1, 2, 3), (8, 8, 63, 1), (8, 4, 128, 2), (32, 2, 1279, 1)])
def test_decode_rope_append_fused_bit_identical(hq, hkv, ctx, b):
    """hx_attn_decode_rope_append == hx_rope_kv_append + hx_attn_decode_paged, bit for
    bit (q, the appended K/V page slots and the attention output), with per-sequence
    lengths that put the new token at page starts, page ends and mid-page."""
    dt, hd, page = torch.bfloat16, 128, 64
    kc, vc, bt, g = _paged_setup(dt, b, hq, hkv, hd, page, ctx + 1)
    n = (hq + 2 * hkv) * hd
    hist = torch.randn(b * ctx, n, device=DEV, generator=g).to(dt)
    seq = torch.zeros(b, dtype=torch.int32, device=DEV)
    ops.rope_kv_append(hist, torch.empty(b * ctx, hq * hd, device=DEV, dtype=dt), kc, vc, bt, seq, b * ctx, ctx,
                       hq, hkv, hd, 10000.0)
    lens = [max(0, ctx - 64 * i - (i % 3)) for i in range(b)]
    seq.copy_(torch.tensor(lens, dtype=torch.int32))
    new = torch.randn(b, n, device=DEV, generator=g).to(dt)
    ws = torch.zeros(ops.attn_decode_workspace(b, hq, hkv, hd, ctx + 1) // 4 + 64, dtype=torch.int32, device=DEV)
    k2, v2 = kc.clone(), vc.clone()
    q = torch.empty(b, hq * hd, device=DEV, dtype=dt)
    o_sep = torch.empty(b, hq * hd, device=DEV, dtype=dt)
    ops.rope_kv_append(new, q, kc, vc, bt, seq, b, 0, hq, hkv, hd, 10000.0)
    ops.attn_decode(q, kc, vc, bt, seq, o_sep, b, hq, hkv, hd, ctx + 1, ws)
    o_fused = torch.empty_like(o_sep)
    ops.attn_decode_rope_append(new, k2, v2, bt, seq, o_fused, b, hq, hkv, hd, ctx + 1, 10000.0, ws)
    torch.cuda.synchronize()
    assert torch.equal(k2, kc) and torch.equal(v2, vc)
    assert torch.equal(o_fused, o_sep)


@pytest.mark.parametrize("b,hq,hkv,ctx", [(32, 32, 4, 1100), (16, 16, 2, 700), (12, 32, 4, 500), (8, 64, 8, 1279)])
def test_decode_attention_cluster_split_combine(b, hq, hkv, ctx):
    """(batch, kv-head) pair counts that give 2-8 KV splits: the splits of a
    pair run as one thread-block cluster and combine over DSMEM. Checked
    against the torch reference, and fused (RoPE + append) == separate."""
    dt, hd, page = torch.bfloat16, 128, 64
    kc, vc, bt, g = _paged_setup(dt, b, hq, hkv, hd, page, ctx + 1)
    n = (hq + 2 * hkv) * hd
    seq = torch.zeros(b, dtype=torch.int32, device=DEV)
    hist = torch.randn(b * ctx, n, device=DEV, generator=g).to(dt)
    ops.rope_kv_append(hist, torch.empty(b * ctx, hq * hd, device=DEV, dtype=dt), kc, vc, bt, seq, b * ctx, ctx,
                       hq, hkv, hd, 10000.0)
    seq.copy_(torch.tensor([max(1, ctx - 37 * i) for i in range(b)], dtype=torch.int32))
    kr, vr = kc.clone(), vc.clone()
    new = torch.randn(b, n, device=DEV, generator=g).to(dt)
    q, qr = (torch.empty(b, hq * hd, device=DEV, dtype=dt) for _ in range(2))
    ws = torch.zeros(ops.attn_decode_workspace(b, hq, hkv, hd, ctx + 1) // 4 + 64, dtype=torch.int32, device=DEV)
    k2, v2 = kc.clone(), vc.clone()
    ops.rope_kv_append(new, q, kc, vc, bt, seq, b, 0, hq, hkv, hd, 10000.0)
    ref.rope_kv_append(new, qr, kr, vr, bt, seq, b, 0, hq, hkv, hd, 10000.0)
    o = torch.empty(b, hq * hd, device=DEV, dtype=dt)
    want = torch.empty(b, hq * hd, device=DEV)
    ops.attn_decode(q, kc, vc, bt, seq, o, b, hq, hkv, hd, ctx + 1, ws)
    ref.attn_decode(qr, kr, vr, bt, seq, want, b, hq, hkv, hd, ctx + 1)
    o_fused = torch.empty_like(o)
    ops.attn_decode_rope_append(new, k2, v2, bt, seq, o_fused, b, hq, hkv, hd, ctx + 1, 10000.0, ws)
    torch.cuda.synchronize()
    assert rel_err(o, want) < 2e-2
    assert torch.equal(o_fused, o)


def test_decode_rope_append_fused_unsupported_shapes():
    assert not ops.decode_rope_fusable(torch.float32, 128, 64, 8, 8)
    assert not ops.decode_rope_fusable(torch.bfloat16, 64, 64, 8, 8)
    assert not ops.decode_rope_fusable(torch.bfloat16, 128, 16, 8, 8)
    dt = torch.bfloat16
    kc, vc, bt, _ = _paged_setup(dt, 1, 4, 4, 128, 16, 32)
    qkv = torch.zeros(1, 12 * 128, device=DEV, dtype=dt)
    seq = torch.zeros(1, dtype=torch.int32, device=DEV)
    with pytest.raises(ops.HxError):
        ops.attn_decode_rope_append(qkv, kc, vc, bt, seq, torch.empty(1, 4 * 128, device=DEV, dtype=dt),
                                    1, 4, 4, 128, 32, 10000.0)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("hq,hkv,hd,s", [(8, 8, 32, 64), (4, 4, 128, 200), (8, 2, 128, 130), (2, 2, 64, 1),
                                          (4, 4, 64, 257), (2, 1, 128, 64), (1, 1, 128, 513)])
def test_prefill_attention(dt, hq, hkv, hd, s):
    b, page = 2, 16
    kc, vc, bt, g = _paged_setup(dt, b, hq, hkv, hd, page, s)
    seq = torch.zeros(b, dtype=torch.int32, device=DEV)
    n = (hq + 2 * hkv) * hd
    qkv = torch.randn(b * s, n, device=DEV, generator=g).to(dt)
    q = torch.empty(b * s, hq * hd, device=DEV, dtype=dt)
    ops.rope_kv_append(qkv, q, kc, vc, bt, seq, b * s, s, hq, hkv, hd, 10000.0)
    o = torch.empty(b * s, hq * hd, device=DEV, dtype=dt)
    ops.attn_prefill(q, kc, vc, bt, seq, o, b, s, hq, hkv, hd)
    want = torch.empty(b * s, hq * hd, device=DEV)
    ref.attn_prefill(q, kc, vc, bt, seq, want, b, s, hq, hkv, hd)
    torch.cuda.synchronize()
    assert rel_err(o, want) < (2e-5 if dt == torch.float32 else 2e-2)


@pytest.mark.parametrize("b,s,hq,hkv", [(2, 128, 4, 4), (2, 256, 8, 2), (1, 512, 8, 1), (3, 384, 16, 8)])
def test_prefill_attention_tcgen05(b, s, hq, hkv):
    """tcgen05 causal prefill attention (TMEM S/PV accumulators, P through smem)
    against the torch fp32 reference on the same paged K and roped q."""
    dt, hd, page = torch.bfloat16, 128, 64
    kc, vc, bt, g = _paged_setup(dt, b, hq, hkv, hd, page, s, seed=3)
    seq = torch.zeros(b, dtype=torch.int32, device=DEV)
    qkv = torch.randn(b * s, (hq + 2 * hkv) * hd, device=DEV, generator=g).to(dt)
    q = torch.empty(b * s, hq * hd, device=DEV, dtype=dt)
    ops.rope_kv_append(qkv, q, kc, vc, bt, seq, b * s, s, hq, hkv, hd, 10000.0)
    vt = torch.empty(b * hkv * hd * s, device=DEV, dtype=dt)
    ops.prefill_vt(qkv, vt, b, s, hq, hkv, hd)
    o = torch.empty(b * s, hq * hd, device=DEV, dtype=dt)
    ops.attn_prefill_tc(q, kc, vt, bt, o, b, s, hq, hkv, hd)
    want = torch.empty(b * s, hq * hd, device=DEV)
    ref.attn_prefill(q, kc, vc, bt, seq, want, b, s, hq, hkv, hd)
    # vt is V transposed per (sequence, kv head)
    v = qkv.view(b, s, hq + 2 * hkv, hd)[:, :, hq + hkv:].float()
    assert torch.equal(vt.view(b, hkv, hd, s).float(), v.permute(0, 2, 3, 1))
    torch.cuda.synchronize()
    assert rel_err(o, want) < 2e-2


@pytest.mark.parametrize("b,hq,hkv,hidden,ctx", [(8, 32, 32, 4096, 575), (32, 16, 2, 8192, 1100), (8, 20, 20, 5120, 600),
                                                (32, 32, 4, 8192, 700), (4, 8, 8, 2048, 130)])
def test_deferred_qkv_into_attention_bit_identical(b, hq, hkv, hidden, ctx):
    """QKV as a deferred stream-K GEMM (fp32 partial slots, no fix-up) whose split
    tiles the attention prologue reduces (hx_attn_decode_rope_append_sk) ==
    hx_linear (bf16 qkv, in-kernel fix-up) + hx_attn_decode_rope_append, bit for
    bit: attention output and the appended K/V page slots. Shapes: 7B, 70B TP=4,
    13B TP=2, 70B TP=2, small."""
    dt, hd, page = torch.bfloat16, 128, 64
    kc, vc, bt, g = _paged_setup(dt, b, hq, hkv, hd, page, ctx + 1)
    n = (hq + 2 * hkv) * hd
    hist = torch.randn(b * ctx, n, device=DEV, generator=g).to(dt)
    seq = torch.zeros(b, dtype=torch.int32, device=DEV)
    ops.rope_kv_append(hist, torch.empty(b * ctx, hq * hd, device=DEV, dtype=dt), kc, vc, bt, seq, b * ctx, ctx,
                       hq, hkv, hd, 10000.0)
    seq.copy_(torch.tensor([max(1, ctx - 61 * i) for i in range(b)], dtype=torch.int32))
    w = ops.PackedWeight((torch.randn(n, hidden, device=DEV, generator=g) * 0.02).bfloat16())
    x = torch.randn(b, hidden, device=DEV, generator=g).bfloat16()
    lin_ws = torch.zeros(ops.linear_workspace(dt, b, n, hidden) // 4 + 64, dtype=torch.int32, device=DEV)
    attn_ws = torch.zeros(ops.attn_decode_workspace(b, hq, hkv, hd, ctx + 1) // 4 + 64, dtype=torch.int32,
                          device=DEV)
    k2, v2 = kc.clone(), vc.clone()
    qkv = torch.empty(b, n, device=DEV, dtype=dt)
    o_ref = torch.empty(b, hq * hd, device=DEV, dtype=dt)
    ops.linear(w, x, qkv, b, lin_ws)
    ops.attn_decode_rope_append(qkv, kc, vc, bt, seq, o_ref, b, hq, hkv, hd, ctx + 1, 10000.0, attn_ws)
    qkv32 = torch.full((b, n), float("nan"), device=DEV)
    o_def = torch.empty_like(o_ref)
    for _ in range(2):   # the second call reuses the re-armed tickets
        ops.linear(w, x, qkv32, b, lin_ws, defer_reduce=True)
        ops.attn_decode_rope_append_sk(qkv32, lin_ws, hidden, k2, v2, bt, seq, o_def, b, hq, hkv, hd, ctx + 1,
                                       10000.0, attn_ws)
        torch.cuda.synchronize()
        assert torch.equal(k2, kc) and torch.equal(v2, vc)
        assert torch.equal(o_def, o_ref)
