"""CPU fp32 ORACLE for the asymmetric TP/PP decoder data path -- TEST
INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline -- never as the product path.

Parity anchor. The reference (heteroplan) has no data-path implementation
(reference ``SPEC.md:8,579``); the layer math is pinned by the paper:
  * prefill layer: x_Q, x_K, x_V = x.w_Q/K/V; softmax(x_Q x_K^T / sqrt(d)) x_V w_O
    + x; MLP(x_Out) + x_Out -- ``PAPER.md:121-135``
  * decode: concat the new token's K/V to the cache, then the same layer math
    for one token -- ``PAPER.md:137-151``
  * TP = column/row split with 2 all-reduces per layer; PP = stage j sends
    its activation to stage j+1 -- ``PAPER.md:158-160, 197``
with Llama-2 specifics (RMSNorm eps, rotate-half RoPE theta 1e4, SwiGLU, GQA,
sqrt(head_dim) scaling, untied lm_head) pinned against HF transformers 5.5
``LlamaForCausalLM`` by ``tests/golden/make_golden.py`` (fixtures committed
in ``tests/golden/tiny_hf.npz``). Generation follows HF ``max_new_tokens``
semantics: the prefill emits token 1, then ``s_out - 1`` decode steps
(SURVEY Appendix B #2).

Everything is float32 numpy. ``Oracle.generate`` runs the unsharded model;
``sharded_generate`` runs the same math split per plan stage and TP rank,
summing partials in rank order, to pin the sharding the engine uses.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    x = x.astype(F32)
    var = np.mean(x * x, axis=-1, keepdims=True, dtype=F32)
    return (x * (F32(1.0) / np.sqrt(var + F32(eps)))).astype(F32) * w


def rope_tables(head_dim: int, theta: float, positions: np.ndarray):
    """HF LlamaRotaryEmbedding (default rope): inv_freq in fp32, angle = pos*inv_freq."""
    inv_freq = (F32(1.0) / (F32(theta) ** (np.arange(0, head_dim, 2, dtype=np.int64)
                                           .astype(F32) / F32(head_dim)))).astype(F32)
    ang = positions.astype(F32)[..., None] * inv_freq          # [..., hd/2]
    ang = np.concatenate([ang, ang], axis=-1)
    return np.cos(ang).astype(F32), np.sin(ang).astype(F32)


def apply_rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """x [..., hd]; rotate_half(x) = cat(-x2, x1)."""
    h = x.shape[-1] // 2
    rot = np.concatenate([-x[..., h:], x[..., :h]], axis=-1)
    return (x * cos + rot * sin).astype(F32)


def silu(x):
    return (x / (F32(1.0) + np.exp(-x))).astype(F32)


def lin(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """x[..., K] @ w[N, K]^T computed as (w @ x2^T)^T: OpenBLAS streams the
    row-major weight once instead of a slow transposed-B path for skinny x."""
    x2 = np.ascontiguousarray(x.reshape(-1, x.shape[-1]), dtype=F32)
    return np.ascontiguousarray((w @ x2.T).T).reshape(*x.shape[:-1], w.shape[0])


class Cache:
    """Per-layer K/V, [b, kv_heads, t, hd] fp32 (a contiguous stand-in for pages)."""

    def __init__(self):
        self.k = {}
        self.v = {}


def attention(q, k, v, causal_offset):
    """q [b, hq, s, hd]; k, v [b, hkv, t, hd]; query i sees keys <= i + offset."""
    b, hq, s, hd = q.shape
    hkv, t = k.shape[1], k.shape[2]
    g = hq // hkv
    k = np.repeat(k, g, axis=1)
    v = np.repeat(v, g, axis=1)
    scores = np.matmul(q, np.swapaxes(k, -1, -2)).astype(F32) * F32(1.0 / np.sqrt(hd))
    qi = np.arange(s)[:, None] + causal_offset
    kj = np.arange(t)[None, :]
    scores = np.where(kj <= qi, scores, F32(-np.inf))
    m = scores.max(axis=-1, keepdims=True)
    p = np.exp(scores - m).astype(F32)
    p /= p.sum(axis=-1, keepdims=True)
    return np.matmul(p, v).astype(F32)


class Oracle:
    """Unsharded fp32 Llama forward with a KV cache.

    ``act_bf16=True`` additionally rounds to bf16 exactly where the bf16-mode
    engine stores bf16 (norm outputs, qkv, roped q/k and v in the cache,
    attention output, gate/up and SwiGLU outputs); the residual stream, the
    row-parallel outputs and logits stay fp32 as in the engine."""

    def __init__(self, cfg, weights, act_bf16=False):
        self.cfg = cfg
        self.w = weights
        self.r = bf16_round if act_bf16 else (lambda a: a)

    def layer(self, l, x, pos0, cache):
        cfg, lw = self.cfg, self.w["layers"][l]
        b, s, H = x.shape
        hd, hq, hkv = cfg.head_dim, cfg.num_heads, cfg.num_kv_heads
        r = self.r
        h = r(rmsnorm(x, lw["ln_attn"], cfg.rms_eps))
        q = r(lin(h, lw["q"])).reshape(b, s, hq, hd).transpose(0, 2, 1, 3)
        k = r(lin(h, lw["k"])).reshape(b, s, hkv, hd).transpose(0, 2, 1, 3)
        v = r(lin(h, lw["v"])).reshape(b, s, hkv, hd).transpose(0, 2, 1, 3)
        cos, sin = rope_tables(hd, cfg.rope_theta, np.arange(pos0, pos0 + s))
        q, k = r(apply_rope(q, cos, sin)), r(apply_rope(k, cos, sin))
        if l in cache.k:
            cache.k[l] = np.concatenate([cache.k[l], k], axis=2)
            cache.v[l] = np.concatenate([cache.v[l], v], axis=2)
        else:
            cache.k[l], cache.v[l] = k, v
        o = r(attention(q, cache.k[l], cache.v[l], pos0))
        o = o.transpose(0, 2, 1, 3).reshape(b, s, hq * hd)
        x = (x + lin(o, lw["o"])).astype(F32)
        h = r(rmsnorm(x, lw["ln_mlp"], cfg.rms_eps))
        a = r(silu(r(lin(h, lw["gate"]))) * r(lin(h, lw["up"])))  # silu in fp32, one rounding
        return (x + lin(a, lw["down"])).astype(F32)

    def logits(self, x_last):
        h = self.r(rmsnorm(x_last, self.w["norm"], self.cfg.rms_eps))
        return lin(h, self.w["lm_head"]).astype(F32)

    def forward(self, ids, pos0, cache):
        x = self.w["embed"][ids].astype(F32)
        for l in range(self.cfg.num_layers):
            x = self.layer(l, x, pos0, cache)
        return self.logits(x[:, -1])

    def generate(self, prompt, s_out, forced=None):
        """Greedy; returns (ids [b, s_out] int32, logits [s_out, b, V] fp32).
        ``forced`` [b, s_out] teacher-forces the fed-back token (bf16 checks)."""
        prompt = np.asarray(prompt)
        b, s_in = prompt.shape
        cache = Cache()
        out_ids, out_logits = [], []
        lg = self.forward(prompt, 0, cache)
        for t in range(s_out):
            nxt = np.argmax(lg, axis=-1).astype(np.int32)
            out_ids.append(nxt)
            out_logits.append(lg)
            if t + 1 == s_out:
                break
            feed = nxt if forced is None else np.asarray(forced)[:, t].astype(np.int32)
            lg = self.forward(feed[:, None], s_in + t, cache)
        return np.stack(out_ids, axis=1), np.stack(out_logits, axis=0)


class ShardedOracle(Oracle):
    """Same math, executed per plan stage and TP rank with explicit partial sums
    (PAPER.md:158-160): column-parallel QKV / gate-up, row-parallel O / down
    whose per-rank partials are summed in rank order (the all-reduce), and a
    vocab-parallel lm_head whose argmax is taken over the concatenated shards.
    ``stages`` = [(tp, (l0, l1)), ...]."""

    def __init__(self, cfg, weights, stages):
        super().__init__(cfg, weights)
        from paper_2311_11514_b200.weights import shard_layer
        self.stages = stages
        self.shards = {}
        for tp, (l0, l1) in stages:
            for l in range(l0, l1):
                self.shards[l] = [shard_layer(cfg, weights["layers"][l], r, tp) for r in range(tp)]

    def layer(self, l, x, pos0, cache):
        cfg = self.cfg
        b, s, H = x.shape
        hd = cfg.head_dim
        shards = self.shards[l]
        tp = len(shards)
        hq, hkv = cfg.num_heads // tp, cfg.num_kv_heads // tp
        partial = []
        h = rmsnorm(x, shards[0]["ln_attn"], cfg.rms_eps)
        cos, sin = rope_tables(hd, cfg.rope_theta, np.arange(pos0, pos0 + s))
        for r, sw in enumerate(shards):
            qkv = lin(h, sw["wqkv"])
            q = qkv[..., :hq * hd].reshape(b, s, hq, hd).transpose(0, 2, 1, 3)
            k = qkv[..., hq * hd:(hq + hkv) * hd].reshape(b, s, hkv, hd).transpose(0, 2, 1, 3)
            v = qkv[..., (hq + hkv) * hd:].reshape(b, s, hkv, hd).transpose(0, 2, 1, 3)
            q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
            key = (l, r)
            if key in cache.k:
                cache.k[key] = np.concatenate([cache.k[key], k], axis=2)
                cache.v[key] = np.concatenate([cache.v[key], v], axis=2)
            else:
                cache.k[key], cache.v[key] = k, v
            o = attention(q, cache.k[key], cache.v[key], pos0)
            o = o.transpose(0, 2, 1, 3).reshape(b, s, hq * hd)
            partial.append(lin(o, sw["wo"]))
        x = (x + _rank_order_sum(partial)).astype(F32)
        h = rmsnorm(x, shards[0]["ln_mlp"], cfg.rms_eps)
        partial = []
        for sw in shards:
            gu = lin(h, sw["wgu"])
            n = gu.shape[-1] // 2
            partial.append(lin(silu(gu[..., :n]) * gu[..., n:], sw["wdown"]))
        return (x + _rank_order_sum(partial)).astype(F32)

    def logits(self, x_last):
        tp = self.stages[-1][0]
        h = rmsnorm(x_last, self.w["norm"], self.cfg.rms_eps)
        V = self.cfg.vocab
        parts = [lin(h, self.w["lm_head"][r * V // tp:(r + 1) * V // tp]) for r in range(tp)]
        return np.concatenate(parts, axis=-1).astype(F32)


def _rank_order_sum(parts):
    acc = parts[0].astype(F32)
    for p in parts[1:]:
        acc = (acc + p).astype(F32)
    return acc


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as fp32 (what the GPU stores)."""
    u = np.ascontiguousarray(x, dtype=F32).view(np.uint32)
    r = ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000))
    return r.view(F32)


def bf16_weights(w: dict) -> dict:
    """The weights exactly as the bf16-mode engine holds them (norm gains kept fp32)."""
    out = {k: (bf16_round(v) if k in ("embed", "lm_head") else v) for k, v in w.items() if k != "layers"}
    out["layers"] = {l: {k: (v if k.startswith("ln_") else bf16_round(v)) for k, v in lw.items()}
                     for l, lw in w["layers"].items()}
    return out


def streamed_teacher_forced(cfg, seed, seq, positions, modes=((True, True), (True, False))):
    """Teacher-forced logits of a full-depth model without holding it in host
    RAM (C2: 7B fp32 is 27 GB): one causal pass over ``seq`` [b, t] (prompt +
    forced tokens), layer by layer, each layer's weights drawn from the same
    seeded streams as ``init_tensor`` (``weights.layer_stream``), used by every
    mode and dropped. Equivalent to prefill + teacher-forced decode steps (the
    layer math is per position except the causal attention; the engine stores
    bf16 at the same points in both phases). ``modes``: (weights rounded to bf16, activations rounded to bf16)
    pairs; returns {mode: logits [len(positions), b, V]}."""
    from paper_2311_11514_b200.weights import init_globals, layer_stream
    seq = np.asarray(seq)
    modes = [tuple(m) for m in modes]
    g32 = init_globals(cfg, seed, ("embed", "norm", "lm_head"))
    gb = {k: (v if k == "norm" else bf16_round(v)) for k, v in g32.items()}
    glob = {True: gb, False: g32}
    xs = {m: glob[m[0]]["embed"][seq].astype(F32) for m in modes}
    for l, lw in layer_stream(cfg, seed, range(cfg.num_layers)):
        w = {False: {"layers": {l: lw}}}
        if any(m[0] for m in modes):
            w[True] = {"layers": {l: {k: (v if k.startswith("ln_") else bf16_round(v)) for k, v in lw.items()}}}
        for m in modes:
            xs[m] = Oracle(cfg, w[m[0]], act_bf16=m[1]).layer(l, xs[m], 0, Cache())
        del w, lw
    pos = list(positions)
    out = {}
    for m in modes:
        o = Oracle(cfg, glob[m[0]], act_bf16=m[1])
        out[m] = np.stack([o.logits(xs[m][:, p]) for p in pos], 0)
    return out
