"""TEST-ONLY stand-in for ``paper_2311_11514_b200.ops`` on CPU tensors.

Implements the same entry points (same arguments, same buffer semantics:
paged KV layout, seq_lens, packed argmax keys) with plain torch fp32 math so
the engine's host logic -- sharding, stage phases, all-reduce placement,
hand-off routing, token return, KV paging -- can be exercised on CPU and
under gloo with several processes. The product path never imports this.
"""

from __future__ import annotations

import torch


def _f(t):
    return t.float()


def embed(ids, table, x, n_tok):
    x[:n_tok] = _f(table)[ids[:n_tok].long()]


def rmsnorm(x, gain, out, n_tok, eps, ldx=None):
    H = gain.shape[0]
    ldx = ldx or H
    flat = x.reshape(-1)
    rows = torch.stack([flat[t * ldx:t * ldx + H] for t in range(n_tok)]) if ldx != H else x[:n_tok]
    var = (rows * rows).mean(-1, keepdim=True)
    out[:n_tok] = (rows * (1.0 / torch.sqrt(var + eps)) * gain).to(out.dtype)


def residual_add_rmsnorm(x, delta, gain, out, n_tok, eps):
    x[:n_tok] += delta[:n_tok]
    if out is not None:
        rmsnorm(x, gain, out, n_tok, eps)


def linear_workspace(dtype, n_tok, n_out, k_dim):
    return 0


def linear(w, x, y, n_tok, workspace=None, accumulate=False):
    r = _f(x[:n_tok]) @ _f(w).T
    if accumulate:
        y[:n_tok, :w.shape[0]] += r
    else:
        y[:n_tok, :w.shape[0]] = r.to(y.dtype)


def swiglu(gu, out, n_tok):
    n = out.shape[-1]
    g, u = _f(gu[:n_tok, :n]), _f(gu[:n_tok, n:2 * n])
    out[:n_tok] = (g / (1.0 + torch.exp(-g)) * u).to(out.dtype)


def _slot(block_table, page, b, pos):
    return int(block_table[b, pos // page]), pos % page


def rope_kv_append(qkv, q_out, k_cache, v_cache, block_table, seq_lens, n_tok, prefill_len, hq, hkv, hd, theta):
    page = k_cache.shape[2]
    half = hd // 2
    inv = 1.0 / (torch.tensor(theta, dtype=torch.float32) **
                 (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    for t in range(n_tok):
        b = t // prefill_len if prefill_len else t
        pos = int(seq_lens[b]) + (t % prefill_len if prefill_len else 0)
        ang = torch.tensor(float(pos), dtype=torch.float32) * inv
        ang = torch.cat([ang, ang])
        c, s = torch.cos(ang).to(qkv.device), torch.sin(ang).to(qkv.device)
        row = _f(qkv[t])
        heads = row[:(hq + hkv) * hd].view(hq + hkv, hd)
        rot = torch.cat([-heads[:, half:], heads[:, :half]], -1)
        roped = heads * c + rot * s
        q_out[t] = roped[:hq].reshape(-1).to(q_out.dtype)
        blk, off = _slot(block_table, page, b, pos)
        k_cache[blk, :, off] = roped[hq:].to(k_cache.dtype)
        v_cache[blk, :, off] = row[(hq + hkv) * hd:].view(hkv, hd).to(v_cache.dtype)


def _gather_kv(cache, block_table, b, n, page):
    out = []
    for p in range(n):
        blk, off = _slot(block_table, page, b, p)
        out.append(_f(cache[blk, :, off]))
    return torch.stack(out, 1)  # [hkv, n, hd]


def attn_decode_workspace(batch, hq, hkv, hd, max_ctx):
    return 0


def attn_decode(q, k_cache, v_cache, block_table, seq_lens, o, batch, hq, hkv, hd, max_ctx, workspace=None):
    page = k_cache.shape[2]
    g = hq // hkv
    for b in range(batch):
        ctx = int(seq_lens[b]) + 1
        K = _gather_kv(k_cache, block_table, b, ctx, page).repeat_interleave(g, 0)
        V = _gather_kv(v_cache, block_table, b, ctx, page).repeat_interleave(g, 0)
        qb = _f(q[b]).view(hq, 1, hd)
        s = (qb @ K.transpose(-1, -2)) / (hd ** 0.5)
        p = torch.softmax(s, -1)
        o[b] = (p @ V).reshape(-1).to(o.dtype)


def attn_prefill(q, k_cache, v_cache, block_table, seq_lens, o, batch, s, hq, hkv, hd):
    page = k_cache.shape[2]
    g = hq // hkv
    for b in range(batch):
        p0 = int(seq_lens[b])
        K = torch.stack([_f(k_cache[_slot(block_table, page, b, p0 + j)[0], :, (p0 + j) % page])
                         for j in range(s)], 1).repeat_interleave(g, 0)
        V = torch.stack([_f(v_cache[_slot(block_table, page, b, p0 + j)[0], :, (p0 + j) % page])
                         for j in range(s)], 1).repeat_interleave(g, 0)
        qb = _f(q[b * s:(b + 1) * s]).view(s, hq, hd).transpose(0, 1)
        sc = (qb @ K.transpose(-1, -2)) / (hd ** 0.5)
        mask = torch.triu(torch.ones(s, s, dtype=torch.bool, device=q.device), 1)
        sc = sc.masked_fill(mask, float("-inf"))
        p = torch.softmax(sc, -1)
        o[b * s:(b + 1) * s] = (p @ V).transpose(0, 1).reshape(s, -1).to(o.dtype)


def advance(seq_lens, batch, n):
    seq_lens[:batch] += n


def _pack(v: float, idx: int) -> int:
    import struct
    bits = struct.unpack("<I", struct.pack("<f", v))[0]
    ordv = (~bits & 0xFFFFFFFF) if bits & 0x80000000 else (bits | 0x80000000)
    ordv ^= 0x80000000
    key = (ordv << 32) | (0xFFFFFFFF - idx)
    return key - (1 << 64) if key >= (1 << 63) else key


def argmax_partial(logits, keys, n_tok, n_cols, vocab_offset):
    for t in range(n_tok):
        i = int(torch.argmax(logits[t, :n_cols]))
        keys[t] = _pack(float(logits[t, i]), i + vocab_offset)


def argmax_finalize(keys, ids, history, step, n_tok, bump=True):
    st = int(step[0]) if history is not None else 0
    for t in range(n_tok):
        lo = int(keys[t]) & 0xFFFFFFFF
        ids[t] = 0xFFFFFFFF - lo
        if history is not None and st < history.shape[1]:
            history[t, st] = ids[t]
    if history is not None and bump:
        step[0] = st + 1
