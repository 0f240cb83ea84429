"""The asymmetric TP/PP stage executor (the runtime the reference only models).

Reference anchors: the plan it executes (``costs.py:43-92``, ``cli.py:95-106``),
the per-layer math (``PAPER.md:114-154``), TP = 2 all-reduces per layer and
PP = per-stage TP degree + uneven layer counts with a stage-to-stage
activation hand-off (``PAPER.md:158-160, 195-197``). The cost model's terms
(``costs.py:106-176``) are what each piece below replaces with real work.

Structure (one process per GPU in production; see ``comm.py`` for the
single-process emulation used by parity tests):

* ``RankExecutor`` -- one (stage, TP rank): its weight shards, paged KV cache
  for its layers, static activation buffers, and the kernel sequence of a
  layer split into the phases between collectives;
* ``StageDriver`` -- runs the ranks of one stage in lockstep through
  attention -> all-reduce -> MLP -> all-reduce, the final norm + vocab-parallel
  lm_head + cross-rank argmax on the last stage, and the stage hand-off;
* ``Engine`` -- the request API (``generate`` for a ``TaskSpec``-shaped batch,
  ``service_time`` for the reference's service-time seam); captures each
  stage's decode step in a CUDA graph.

All arithmetic happens in ``ops`` (the C-ABI kernels); this module only moves
pointers, issues collectives and sequences launches.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import ops as _ops
from .comm import make_comm
from .config import LlamaConfig
from .plan import GlobalAssignment, InputError, TaskSpec
from .topology import Role, pipeline_roles, role_of
from .weights import _CODES, LAYER_TENSORS, init_globals, layer_stream, shard_layer, tensor_shape

DTYPES = {"bf16": torch.bfloat16, "fp32": torch.float32}


# --------------------------------------------------------------------- weights
def _device_tensor(cfg, seed, name, layer, device):
    """Synthetic weights generated on the device (fast path for large models):
    normal(0, 0.02) (+1 for norm gains) from a per-tensor torch generator."""
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + (layer + 1) * 1009 + _CODES[name]) & 0x7FFFFFFFFFFFFFFF)
    t = torch.randn(tensor_shape(cfg, name), generator=g, device=device, dtype=torch.float32)
    t.mul_(0.02)
    if name in ("norm", "ln_attn", "ln_mlp"):
        t.add_(1.0)
    return t


def _shard_device(cfg, lw, r, tp):
    H = cfg.hidden_dim
    hd = cfg.head_dim
    qn, kn, In = cfg.num_heads * hd // tp, cfg.num_kv_heads * hd // tp, cfg.intermediate // tp
    return {
        "wqkv": torch.cat([lw["q"][r * qn:(r + 1) * qn], lw["k"][r * kn:(r + 1) * kn],
                           lw["v"][r * kn:(r + 1) * kn]], 0),
        "wo": lw["o"][:, r * qn:(r + 1) * qn],
        "wgu": torch.cat([lw["gate"][r * In:(r + 1) * In], lw["up"][r * In:(r + 1) * In]], 0),
        "wdown": lw["down"][:, r * In:(r + 1) * In],
        "ln_attn": lw["ln_attn"], "ln_mlp": lw["ln_mlp"],
    }


def load_rank_weights(cfg: LlamaConfig, role: Role, dtype: torch.dtype, device, seed: int = 0,
                      source: str = "host") -> dict:
    """Weight shards for one role (see ``load_weights``)."""
    return load_weights(cfg, [role], dtype, device, seed, source)[role.device]


def load_weights(cfg: LlamaConfig, roles, dtype: torch.dtype, device, seed: int = 0,
                 source: str = "host") -> dict:
    """Weight shards for the given roles, ``{role.device: shards}``. Each layer
    is drawn once and sharded for every local TP rank that owns it.
    ``source='host'`` draws the bit-exact numpy streams the CPU oracle uses
    (threaded, ``weights.layer_stream``); ``'device'`` generates on the GPU
    (same distribution, different bits) for throughput runs of large models."""
    out = {r.device: {"layers": []} for r in roles}

    def put(x, keep_fp32=False):
        t = torch.as_tensor(x) if isinstance(x, np.ndarray) else x
        return t.to(device=device, dtype=torch.float32 if keep_fp32 else dtype).contiguous()

    owners = {}
    for r in roles:
        for l in range(*r.layers):
            owners.setdefault(l, []).append(r)
    layers = sorted(owners)
    if source == "host":
        stream = layer_stream(cfg, seed, layers)
    else:
        stream = ((l, {n: _device_tensor(cfg, seed, n, l, device) for n in LAYER_TENSORS}) for l in layers)
    for l, lw in stream:
        for r in owners[l]:
            sh = shard_layer(cfg, lw, r.tp_rank, r.tp) if source == "host" else _shard_device(cfg, lw, r.tp_rank, r.tp)
            out[r.device]["layers"].append({k: put(v, keep_fp32=k.startswith("ln_")) for k, v in sh.items()})
            del sh
        del lw
    want = sorted({n for r in roles for n in (["embed"] if r.is_first else []) + (["norm", "lm_head"] if r.is_last else [])})
    glob = init_globals(cfg, seed, want) if source == "host" else \
        {n: _device_tensor(cfg, seed, n, -1, device) for n in want}
    for r in roles:
        if r.is_first:
            out[r.device]["embed"] = put(glob["embed"])
        if r.is_last:
            out[r.device]["norm"] = put(glob["norm"], keep_fp32=True)
            vr = cfg.vocab // r.tp
            out[r.device]["lm_head"] = put(glob["lm_head"][r.tp_rank * vr:(r.tp_rank + 1) * vr])
    return out


# --------------------------------------------------------------------- KV cache
class PagedKVCache:
    """Paged K/V for one rank's layers: ``k[layer]`` is
    [num_blocks, kv_heads_rank, page, head_dim]. Blocks are handed out from a
    free list; sequence b's table is interleaved across the pool so the
    kernels' block indirection is always exercised (reference memory term:
    ``costs.py:168-176``)."""

    def __init__(self, n_layers, batch, max_tokens, hkv, hd, page, dtype, device):
        self.page = page
        self.max_blocks = math.ceil(max_tokens / page)
        self.num_blocks = batch * self.max_blocks
        shape = (n_layers, self.num_blocks, hkv, page, hd)
        self.k = torch.zeros(shape, dtype=dtype, device=device)
        self.v = torch.zeros(shape, dtype=dtype, device=device)
        self.block_table = torch.zeros(batch, self.max_blocks, dtype=torch.int32, device=device)
        self.seq_lens = torch.zeros(batch, dtype=torch.int32, device=device)
        self.free = list(range(self.num_blocks))
        self.owned: list[int] = []
        self.batch = batch

    def assign(self, batch: int, tokens: int):
        """Allocate ceil(tokens / page) blocks per sequence; reset lengths."""
        self.release()
        need = math.ceil(tokens / self.page)
        if need > self.max_blocks or batch > self.batch:
            raise InputError(f"request needs {need} blocks/seq x {batch}; cache holds "
                             f"{self.max_blocks} x {self.batch}")
        table = np.zeros((self.batch, self.max_blocks), dtype=np.int32)
        for i in range(need):
            for b in range(batch):
                blk = self.free.pop(0)
                table[b, i] = blk
                self.owned.append(blk)
        self.block_table.copy_(torch.from_numpy(table))
        self.seq_lens.zero_()

    def release(self):
        self.free.extend(self.owned)
        self.free.sort()
        self.owned = []

    def nbytes(self) -> int:
        return 2 * self.k.numel() * self.k.element_size()


# --------------------------------------------------------------------- executor
class RankExecutor:
    """One (stage, TP rank) of the pipeline: weights, KV pages, buffers, kernels."""

    def __init__(self, cfg: LlamaConfig, role: Role, dtype: torch.dtype, batch: int, max_prompt: int,
                 max_out: int, device, weights: dict, kernels=None, page_size: int = 64,
                 pack_weights: bool = True, defer_reduce: bool = True):
        self.cfg, self.role, self.dtype, self.device = cfg, role, dtype, torch.device(device)
        self.k = kernels or _ops
        self.w = weights
        # decode RoPE + KV append inside the TMA attention kernel (bit-identical to
        # the separate kernels); HX_FUSE_ROPE_ATTN=0 selects rope_kv_append + attn_decode
        self.rope_in_attn = (self.device.type == "cuda" and self.k is _ops
                             and _ops.decode_rope_fusable(dtype, cfg.head_dim, page_size, cfg.num_heads // role.tp,
                                                          cfg.num_kv_heads // role.tp)
                             and os.environ.get("HX_FUSE_ROPE_ATTN", "1") != "0")
        if pack_weights and dtype == torch.bfloat16 and self.device.type == "cuda":
            # tile-contiguous layout for the weight-streaming GEMM (hx_pack_weight)
            for lw in weights["layers"]:
                for name in ("wqkv", "wo", "wgu", "wdown"):
                    lw[name] = _ops.PackedWeight(lw[name])
            if "lm_head" in weights:
                weights["lm_head"] = _ops.PackedWeight(weights["lm_head"])
            torch.cuda.synchronize(self.device)
        tp = role.tp
        self.hq, self.hkv = cfg.num_heads // tp, cfg.num_kv_heads // tp
        self.hd = cfg.head_dim
        self.inter = cfg.intermediate // tp
        self.vr = cfg.vocab // tp
        self.qkv_n = (self.hq + 2 * self.hkv) * self.hd
        self.batch, self.max_prompt, self.max_out = batch, max_prompt, max_out
        self.cur_b = batch        # sequences of the request in flight (<= batch)
        self.max_ctx = max_prompt + max_out
        self.n_layers = role.layers[1] - role.layers[0]
        H = cfg.hidden_dim
        T = batch * max_prompt
        dev, act = self.device, dtype
        z = lambda *s, dt=act: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
        self.x = z(T, H, dt=torch.float32)
        self.h = z(T, H)
        self.qkv = z(T, self.qkv_n)
        self.q = z(T, self.hq * self.hd)
        self.attn = z(T, self.hq * self.hd)
        self.proj = z(T, H, dt=torch.float32)
        self.gu = z(T, 2 * self.inter)
        self.a = z(T, self.inter)
        self.kv = PagedKVCache(self.n_layers, batch, self.max_ctx, self.hkv, self.hd, page_size, dtype, dev)
        self.ids = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.prompt = torch.zeros(T, dtype=torch.int32, device=dev)
        if role.is_last:
            self.hl = z(batch, H)
            self.logits = z(batch, self.vr, dt=torch.float32)
            self.keys = torch.zeros(batch, dtype=torch.int64, device=dev)
            self.history = torch.zeros(batch, max_out, dtype=torch.int32, device=dev)
            self.step = torch.zeros(1, dtype=torch.int32, device=dev)
        # decode-shaped split-K / split-KV scratch (prefill uses none)
        ws = 0
        if dev.type == "cuda":
            for n_out, kd in ((self.qkv_n, H), (H, self.hq * self.hd), (2 * self.inter, H),
                              (H, self.inter), (self.vr, H)):
                ws = max(ws, self.k.linear_workspace(dtype, batch, n_out, kd))
            self.attn_ws_bytes = self.k.attn_decode_workspace(batch, self.hq, self.hkv, self.hd, self.max_ctx)
        else:
            self.attn_ws_bytes = 0
        self.lin_ws = torch.zeros(max(ws, 256) // 4 + 64, dtype=torch.int32, device=dev)
        self.defer = (tp == 1 and dtype == torch.bfloat16 and dev.type == "cuda" and self.k is _ops
                      and defer_reduce)
        self._defer_now = False
        self.par = None          # ops.PeerAllReduce when TP>1 ranks run in separate processes
        self.stream = None       # this emulated rank's stream (Engine(local_peer=True))
        self._peer_now = False
        self._decode_now = False
        self.attn_ws = torch.zeros(max(self.attn_ws_bytes, 256) // 4 + 64, dtype=torch.int32, device=dev)
        # decode QKV GEMM without its split-K fix-up tail: partial tiles are reduced
        # in the attention prologue (bit-identical); HX_DEFER_QKV=0 disables
        self.defer_qkv = self.rope_in_attn and os.environ.get("HX_DEFER_QKV", "1") != "0"
        self.defer_ar = os.environ.get("HX_DEFER_AR", "1") != "0"   # see _peer_defer
        self.qkv32 = z(batch, self.qkv_n, dt=torch.float32) if self.defer_qkv else None
        # tcgen05 prefill attention (default; HX_PREFILL_TC=0 selects the mma.sync
        # kernel): needs V transposed per (sequence, kv head) -- a prefill-only scratch
        self.tc_prefill = (os.environ.get("HX_PREFILL_TC", "1") == "1" and dtype == torch.bfloat16
                           and dev.type == "cuda" and self.k is _ops and self.hd == 128 and page_size == 64)
        self.vt = z(batch * max_prompt * self.hkv * self.hd) if self.tc_prefill else None
        # decode gate/up GEMM leaves split tiles as fp32 partials; the SwiGLU
        # kernel reduces them (no fix-up tail in the GEMM). Worth it when the
        # 128-row tiles are few enough that stream-K splits most of them
        # (< 2 per SM): 7B -0.6%, 70B TP=4 -1.6%, 70B TP=1 (448 tiles) +0.5%.
        # HX_DEFER_GU=0 / 1 forces it off / on.
        env = os.environ.get("HX_DEFER_GU")
        few_tiles = 2 * self.inter // 128 < 2 * 148
        self.defer_gu = (dtype == torch.bfloat16 and dev.type == "cuda" and self.k is _ops
                         and (env == "1" or (env is None and few_tiles)))
        self.gu32 = z(batch, 2 * self.inter, dt=torch.float32) if self.defer_gu else None
        self._x_full = self.x
        self.bt, self.sl = self.kv.block_table, self.kv.seq_lens   # the current micro-batch's sequences

    def window(self, seq0: int, seqs: int, seq_len: int):
        """Point the residual stream and the KV tables at sequences
        [seq0, seq0 + seqs) of a prefill (micro-batch); ``window(0, 0, 0)``
        restores the whole batch."""
        if seqs == 0:
            self.x, self.bt, self.sl = self._x_full, self.kv.block_table, self.kv.seq_lens
            return
        self.x = self._x_full[seq0 * seq_len:(seq0 + seqs) * seq_len]
        self.bt = self.kv.block_table[seq0:seq0 + seqs]
        self.sl = self.kv.seq_lens[seq0:seq0 + seqs]

    # ---- phases of layer li (local index) between the two all-reduces
    def attn_block(self, li: int, n_tok: int, prefill_len: int):
        k, cfg, lw = self.k, self.cfg, self.w["layers"][li]
        if li == 0:  # input norm of the stage's first layer (x arrived raw)
            k.rmsnorm(self.x, lw["ln_attn"], self.h, n_tok, cfg.rms_eps)
        kc, vc = self.kv.k[li], self.kv.v[li]
        pf = self._l2pf(prefill_len)
        if self.defer_qkv and not prefill_len and n_tok <= 64:  # decode: split-K reduced by the attention kernel
            k.linear(lw["wqkv"], self.h, self.qkv32, n_tok, self.lin_ws, defer_reduce=True, **pf)
            k.attn_decode_rope_append_sk(self.qkv32, self.lin_ws, cfg.hidden_dim, kc, vc, self.bt, self.sl, self.attn,
                                         n_tok, self.hq, self.hkv, self.hd, self.max_ctx, cfg.rope_theta, self.attn_ws)
        elif self.rope_in_attn and not prefill_len:  # decode: RoPE + KV append inside the attention kernel
            k.linear(lw["wqkv"], self.h, self.qkv, n_tok, self.lin_ws, **pf)
            k.attn_decode_rope_append(self.qkv, kc, vc, self.bt, self.sl, self.attn, n_tok,
                                      self.hq, self.hkv, self.hd, self.max_ctx, cfg.rope_theta, self.attn_ws)
        else:
            k.linear(lw["wqkv"], self.h, self.qkv, n_tok, self.lin_ws)
            k.rope_kv_append(self.qkv, self.q, kc, vc, self.bt, self.sl, n_tok,
                             prefill_len, self.hq, self.hkv, self.hd, cfg.rope_theta)
        if prefill_len and self.tc_prefill and prefill_len % 128 == 0:
            nb = n_tok // prefill_len
            k.prefill_vt(self.qkv, self.vt, nb, prefill_len, self.hq, self.hkv, self.hd)
            k.attn_prefill_tc(self.q, kc, self.vt, self.bt, self.attn, nb, prefill_len, self.hq, self.hkv, self.hd)
        elif prefill_len:
            k.attn_prefill(self.q, kc, vc, self.bt, self.sl, self.attn,
                           n_tok // prefill_len, prefill_len, self.hq, self.hkv, self.hd)
        elif not self.rope_in_attn:
            k.attn_decode(self.q, kc, vc, self.bt, self.sl, self.attn, n_tok,
                          self.hq, self.hkv, self.hd, self.max_ctx, self.attn_ws)
        # TP=1 decode: the O/down GEMMs leave split tiles as partials and the
        # residual+norm kernel that consumes them does the reduction
        self._defer_now = (self.defer or self._peer_defer()) and not prefill_len
        self._decode_now = not prefill_len
        # TP>1 decode: the partial goes straight into this rank's NVLink-visible slot
        self._peer_now = self.par is not None and not prefill_len
        self._linear(lw["wo"], self.attn, self._partial_out(2 * li), n_tok)   # row-parallel partial

    def _peer_defer(self) -> bool:
        """TP>1 decode over the push all-reduce: the O/down GEMMs leave split
        tiles as partials and the all-reduce kernel reduces them while it reads
        the row (bit-identical; HX_DEFER_AR=0 keeps the in-GEMM fix-up)."""
        return (self.defer_ar and self.par is not None and self.par.mode == "push" and self.k is _ops
                and self.dtype == torch.bfloat16)

    def _l2pf(self, prefill_len) -> dict:
        """GEMMs that follow the NVLink all-reduce (TP>1 decode) prefetch extra
        weight tiles into L2 while the all-reduce is latency-bound (measured:
        -0.45 ms per 40-layer TP=2 step; it slows back-to-back TP=1 GEMMs)."""
        return {"l2_prefetch": True} if (self.par is not None and not prefill_len) else {}

    def _partial_out(self, site):
        return self.par.slot(site) if self._peer_now else self.proj

    def _linear(self, w, x, y, n_tok):
        if self._defer_now:
            self.k.linear(w, x, y, n_tok, self.lin_ws, defer_reduce=True)
        else:
            self.k.linear(w, x, y, n_tok, self.lin_ws)

    def _add_norm(self, k_dim, gain, out, n_tok, site):
        if self._peer_now:      # all-reduce over peer memory + residual + RMSNorm, one kernel
            if self._defer_now:  # ... with the split-K reduction of the deferred O/down GEMM
                self.par.allreduce_residual_rmsnorm(self.x, site, gain, out, n_tok, self.cfg.rms_eps,
                                                    gemm_ws=self.lin_ws, k_dim=k_dim)
            else:
                self.par.allreduce_residual_rmsnorm(self.x, site, gain, out, n_tok, self.cfg.rms_eps)
        elif self._defer_now:   # TP=1: split-K reduction inside the residual+norm kernel
            self.k.splitk_residual_rmsnorm(self.x, self.proj, self.lin_ws, n_tok, k_dim, gain, out,
                                           self.cfg.rms_eps)
        else:                   # proj already all-reduced (NCCL) or TP=1 prefill
            self.k.residual_add_rmsnorm(self.x, self.proj, gain, out, n_tok, self.cfg.rms_eps)

    def mlp_norm(self, li: int, n_tok: int):
        """all-reduce #1 (TP>1 decode: fused into this kernel) + residual + RMSNorm."""
        self._add_norm(self.hq * self.hd, self.w["layers"][li]["ln_mlp"], self.h, n_tok, 2 * li)

    def mlp_block(self, li: int, n_tok: int):
        self.mlp_norm(li, n_tok)
        self.mlp_body(li, n_tok)

    def mlp_body(self, li: int, n_tok: int):
        k, lw = self.k, self.w["layers"][li]
        if self.defer_gu and n_tok <= 64 and self._decode_now:
            k.linear(lw["wgu"], self.h, self.gu32, n_tok, self.lin_ws, defer_reduce=True, **self._l2pf(0))
            k.splitk_swiglu(self.gu32, self.lin_ws, n_tok, self.cfg.hidden_dim, self.a)
        else:
            k.linear(lw["wgu"], self.h, self.gu, n_tok, self.lin_ws, **self._l2pf(0))
            k.swiglu(self.gu, self.a, n_tok)
        self._linear(lw["wdown"], self.a, self._partial_out(2 * li + 1), n_tok)   # row-parallel partial

    def post_block(self, li: int, n_tok: int):
        nxt = self.w["layers"][li + 1]["ln_attn"] if li + 1 < self.n_layers else None
        self._add_norm(self.inter, nxt, self.h if nxt is not None else None, n_tok, 2 * li + 1)

    def head(self, prefill_len: int):
        """final norm on each sequence's last row + vocab-parallel lm_head + local argmax."""
        k, H, b = self.k, self.cfg.hidden_dim, self.cur_b
        if prefill_len:
            xs = self.x.view(-1)[(prefill_len - 1) * H:]
            k.rmsnorm(xs, self.w["norm"], self.hl, b, self.cfg.rms_eps, ldx=prefill_len * H)
        else:
            k.rmsnorm(self.x, self.w["norm"], self.hl, b, self.cfg.rms_eps)
        k.linear(self.w["lm_head"], self.hl, self.logits, b, self.lin_ws)
        k.argmax_partial(self.logits, self.keys, b, self.vr, self.role.tp_rank * self.vr)

    def finalize(self):
        self.k.argmax_finalize(self.keys, self.ids, self.history, self.step, self.cur_b, bump=True)


# --------------------------------------------------------------------- driver
class RankStreams:
    """Single-GPU emulation of a multi-GPU decode step with the REAL collective
    kernels (``Engine(..., local_peer=True)``): every emulated rank launches on
    its own CUDA stream and the peer pointers of the NVLink all-reduce and the
    P2P hand-offs are same-device pointers.

    * Work between collectives is serialised across ranks with events, so two
      ranks' persistent GEMMs never compete for the SMs.
    * The all-reduce kernels of a stage wait for the whole chain and are then
      launched on all of its ranks' streams at once: they run concurrently and
      genuinely wait for each other's pushes (the protocol of the multi-GPU
      path; ``tp * n_tok * 4`` CTAs must be co-resident, checked by the engine).
    * A hand-off pull is ordered after its push (no long spin on one GPU).
    Outside ``begin()`` / ``end()`` (the prefill) everything runs on the
    caller's stream."""

    def __init__(self, execs, device):
        for e in execs:
            e.stream = torch.cuda.Stream(device)
        self.active = False
        self.deps = []

    def _event(self, stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        self.last[stream] = ev
        return ev

    def begin(self):
        self.main = torch.cuda.current_stream()
        self.last = {}
        self.deps = [self._event(self.main)]
        self.active = True

    def end(self):
        # join every rank stream's last work (a graph capture needs every fork joined)
        for st, ev in self.last.items():
            if st != self.main:
                self.main.wait_event(ev)
        self.deps, self.active, self.last = [], False, {}

    def serial(self, execs, fn):
        if not self.active:
            for e in execs:
                fn(e)
            return
        for e in execs:
            for ev in self.deps:
                e.stream.wait_event(ev)
            with torch.cuda.stream(e.stream):
                fn(e)
            self.deps = [self._event(e.stream)]

    def concurrent(self, execs, fn):
        if not self.active:
            for e in execs:
                fn(e)
            return
        for e in execs:
            for ev in self.deps:
                e.stream.wait_event(ev)
        evs = []
        for e in execs:
            with torch.cuda.stream(e.stream):
                fn(e)
            evs.append(self._event(e.stream))
        self.deps = evs


class StageDriver:
    """Runs the TP ranks of one stage (all of them when emulated in one
    process, or the single local one under torch.distributed)."""

    def __init__(self, execs: list[RankExecutor], comm, stage: int, sched: RankStreams | None = None):
        self.execs, self.comm, self.stage = execs, comm, stage
        self.role = execs[0].role
        self.tp = self.role.tp
        self.sched = sched

    def _each(self, fn):
        """fn(e) for every local rank (serialised across emulated rank streams)."""
        if self.sched is None:
            for e in self.execs:
                fn(e)
        else:
            self.sched.serial(self.execs, fn)

    def _together(self, fn):
        """fn(e) for every local rank; under RankStreams launched concurrently (collectives)."""
        if self.sched is None:
            for e in self.execs:
                fn(e)
        else:
            self.sched.concurrent(self.execs, fn)

    def _ar(self, n_tok):
        if self.tp > 1 and not self.execs[0]._peer_now:  # peer path reduces inside the next kernel
            self.comm.all_reduce_sum([e.proj[:n_tok] for e in self.execs], self.role.tp_group)

    def embed(self, n_tok: int, prefill: bool):
        self._each(lambda e: e.k.embed(e.prompt if prefill else e.ids, e.w["embed"], e.x, n_tok))

    def layers(self, n_tok: int, prefill_len: int):
        for li in range(self.execs[0].n_layers):
            self._each(lambda e: e.attn_block(li, n_tok, prefill_len))
            self._ar(n_tok)
            self._together(lambda e: e.mlp_norm(li, n_tok))
            self._each(lambda e: e.mlp_body(li, n_tok))
            self._ar(n_tok)
            self._together(lambda e: e.post_block(li, n_tok))
        adv = prefill_len if prefill_len else 1
        self._each(lambda e: e.k.advance(e.sl, e.sl.numel(), adv))

    def head(self, prefill_len: int):
        self._each(lambda e: e.head(prefill_len))
        if self.tp > 1:
            keys = [e.keys for e in self.execs]
            if self.sched is None:
                self.comm.all_reduce_max(keys, self.role.tp_group)
            else:
                self.sched.serial(self.execs[-1:], lambda e: self.comm.all_reduce_max(keys, self.role.tp_group))
        self._each(lambda e: e.finalize())

    def send_hidden(self, n_tok, decode: bool = False):
        def one(e):
            if decode and e.p2p_send:      # NVLink P2P store into each receiver's inbox
                for link in e.p2p_send:
                    link.push(e.x[:n_tok])
                return
            if not decode and e.pf_send:   # prefill micro-batch: flow-controlled NVLink P2P
                for link in e.pf_send:
                    link.push_credit(e.x[:n_tok])
                return
            for dst in e.role.send_to:
                self.comm.send(e.x[:n_tok], e.role.device, dst)
        self._each(one)

    def recv_hidden(self, n_tok, decode: bool = False):
        def one(e):
            if decode and e.p2p_recv is not None:
                e.p2p_recv.pull(e.x[:n_tok])
                return
            if not decode and e.pf_recv is not None:
                e.pf_recv.pull_credit(e.x[:n_tok])
                return
            self.comm.recv(e.x[:n_tok], e.role.recv_from, e.role.device)
        self._each(one)

    def send_ids(self):
        def one(e):
            if e.ids_send:
                for link in e.ids_send:
                    link.push(e.ids)
                return
            for dst in e.role.ids_send_to:
                self.comm.send(e.ids, e.role.device, dst)
        self._each(one)

    def recv_ids(self):
        def one(e):
            if e.ids_recv is not None:
                e.ids_recv.pull(e.ids)
                return
            self.comm.recv(e.ids, e.role.ids_recv_from, e.role.device)
        self._each(one)


# --------------------------------------------------------------------- engine
@dataclass
class GenerateResult:
    ids: np.ndarray                 # [b, s_out] int32
    prefill_s: float                # device time of the prefill (max over local stages)
    decode_s: float                 # device time of the s_out - 1 decode steps
    step_ms: list                   # per decode-step device times (ms)
    logits: np.ndarray | None = None
    launches: int = 0               # hx kernels launched (graph replays included)


class Engine:
    """Serve ``TaskSpec``-shaped batches through one pipeline of a plan.

    ``comm='local'`` emulates every rank of the pipeline in this process on
    ``device`` (parity tests; N=1 benchmarks); ``comm='dist'`` runs the one
    role whose plan device id equals this process's torch.distributed rank
    (torchrun, one process per GPU, NCCL)."""

    def __init__(self, plan: GlobalAssignment, cfg: LlamaConfig, *, dtype: str = "bf16",
                 batch: int, max_prompt: int, max_out: int, pipeline: int = 0, comm: str = "local",
                 device=None, seed: int = 0, weights: str = "host", page_size: int = 64,
                 use_graphs: bool = True, kernels=None, pack_weights: bool = True,
                 peer_allreduce: bool = True, local_peer: bool | None = None):
        if dtype not in DTYPES:
            raise InputError(f"dtype must be one of {sorted(DTYPES)}")
        self.plan, self.cfg, self.dtype = plan, cfg, DTYPES[dtype]
        self.batch, self.max_prompt, self.max_out = batch, max_prompt, max_out
        self.comm = make_comm(comm)
        roles = pipeline_roles(plan, pipeline, cfg)
        self.roles = roles
        if self.comm.kind == "dist":
            rank = self.comm.rank
            pid, me = role_of(plan, rank, cfg)
            if pid != pipeline:
                raise InputError(f"rank {rank} has no role in pipeline {pipeline}")
            local = [me]
            self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        else:
            local = roles
            self.device = torch.device(device) if device is not None else torch.device("cuda", 0)
        self.comm.setup(roles, local)
        self.num_stages = roles[0].num_stages
        self.kernels = kernels or _ops
        if self.device.type == "cuda":
            _ops.load()
        shards = load_weights(cfg, local, self.dtype, self.device, seed, weights)
        execs = [RankExecutor(cfg, r, self.dtype, batch, max_prompt, max_out, self.device, shards.pop(r.device),
                              kernels=self.kernels, page_size=page_size,
                              pack_weights=pack_weights and kernels is None) for r in local]
        peer_allreduce = peer_allreduce and os.environ.get("HX_PEER_AR", "1") != "0"
        native = self.device.type == "cuda" and kernels is None
        # single-GPU emulation that still runs the multi-GPU collective kernels
        # (NVLink all-reduce, P2P hand-offs) -- one stream per emulated rank
        if local_peer is None:
            local_peer = os.environ.get("HX_LOCAL_PEER", "0") == "1"
        self.local_peer = bool(local_peer and self.comm.kind == "local" and native and peer_allreduce)
        if self.local_peer:
            worst = max(r.tp for r in roles) * batch * 4
            if worst > _ops.PEER_AR_CORESIDENT:
                raise InputError(f"local_peer emulation needs tp*batch*4 <= {_ops.PEER_AR_CORESIDENT} co-resident "
                                 f"all-reduce CTAs (got {worst})")
        # all-reduce payload on NVLink: bf16 partials (fp32 sums) halve the bytes in
        # bf16 mode; fp32 mode keeps fp32 partials (north-star fp32 criterion).
        # HX_AR_PAYLOAD=fp32|bf16 overrides.
        payload = os.environ.get("HX_AR_PAYLOAD", "bf16" if self.dtype == torch.bfloat16 else "fp32")
        if payload == "bf16" and (cfg.hidden_dim % 32 or os.environ.get("HX_AR_MODE", "push") == "pull"):
            payload = "fp32"
        self.ar_payload = payload
        if peer_allreduce and self.comm.kind == "dist" and native:
            for e in execs:
                if e.role.tp > 1:  # fused NVLink all-reduce for the decode step
                    e.par = _ops.PeerAllReduce(e.role.tp_rank, e.role.tp, batch, cfg.hidden_dim, 2 * e.n_layers,
                                               self.comm.groups[e.role.tp_group], self.comm.dist, payload=payload)
        elif self.local_peer:
            for j in sorted({r.stage for r in roles}):
                st = sorted((e for e in execs if e.role.stage == j), key=lambda e: e.role.tp_rank)
                if st[0].role.tp > 1:
                    for e, par in zip(st, _ops.PeerAllReduce.local_group(st[0].role.tp, batch, cfg.hidden_dim,
                                                                         2 * st[0].n_layers, payload=payload)):
                        e.par = par
        for e in execs:
            e.p2p_send, e.p2p_recv, e.ids_send, e.ids_recv = [], None, [], None
            e.pf_send, e.pf_recv = [], None
        self._p2p = ((self.comm.kind == "dist" or self.local_peer) and native
                     and self.num_stages > 1 and os.environ.get("HX_P2P", "1") != "0")
        if self._p2p:
            self._setup_p2p(execs)
        self.sched = RankStreams(execs, self.device) if self.local_peer else None
        self.drivers = []
        for j in sorted({r.stage for r in local}):
            self.drivers.append(StageDriver([e for e in execs if e.role.stage == j], self.comm, j, self.sched))
        self.execs = execs
        self.use_graphs = use_graphs and self.device.type == "cuda"
        self._graphs = None
        self._graph_key = None
        self._graph_cache = {}
        self._graph_launches = []
        self._replayed = 0

    def _setup_p2p(self, execs):
        """NVLink P2P links for the decode hand-offs (hidden j -> j+1, ids
        last -> 0), created in one global order so the pairwise handle
        exchanges of every rank line up."""
        links = []
        for r in self.roles:
            links += [("hidden", r.device, dst) for dst in r.send_to]
            links += [("ids", r.device, dst) for dst in r.ids_send_to]
        # the pipelined prefill's hand-offs use their own flow-controlled links
        # (hx_handoff_push/pull_credit), sized for one prefill micro-batch
        if os.environ.get("HX_P2P_PREFILL", "1") != "0":
            links += [("prefill", src, dst) for kind, src, dst in list(links) if kind == "hidden"]
        mb_rows = (self.batch // self.prefill_microbatches(self.batch, self.max_prompt)) * self.max_prompt
        self._pf_rows_cap = mb_rows
        mine = {e.role.device: e for e in execs}
        for kind, src, dst in sorted(links):
            words = {"hidden": self.batch * self.cfg.hidden_dim, "ids": self.batch,
                     "prefill": mb_rows * self.cfg.hidden_dim}[kind]
            if self.local_peer:           # both ends in this process
                link = _ops.P2PLink.local(src, dst, words)
                ends = [(mine[src], True), (mine[dst], False)]
            else:
                me = src if src in mine else dst if dst in mine else None
                if me is None:
                    continue
                link = _ops.P2PLink(src, dst, me, words, self.comm.pairs[(min(src, dst), max(src, dst))],
                                    self.comm.dist)
                ends = [(mine[me], me == src)]
            for e, sender in ends:
                if kind == "prefill":
                    if sender:
                        e.pf_send.append(link)
                    else:
                        e.pf_recv = link
                elif kind == "hidden":
                    if sender:
                        e.p2p_send.append(link)
                    else:
                        e.p2p_recv = link
                elif sender:
                    e.ids_send.append(link)
                else:
                    e.ids_recv = link

    # ---------------------------------------------------------------- steps
    def prefill_microbatches(self, b: int, s: int) -> int:
        """Micro-batches of the prefill: with more than one stage, stage j+1
        prefills micro-batch i while stage j runs i+1 (HexGen App. D pipelining;
        the reference cost model charges the stages' prefill serially,
        costs.py:240-284). Up to 16 micro-batches, each keeping >= 2048 token
        rows for the tensor-core GEMMs; HX_PREFILL_MB overrides."""
        env = os.environ.get("HX_PREFILL_MB")
        if env:
            m = max(1, int(env))
            return m if b % m == 0 else 1
        if self.num_stages == 1:
            return 1
        best = 1
        for m in range(1, 17):   # 70B [2,1,1] b=32 x 1024: m=4 1.75 s, 8 1.51 s, 16 1.45 s
            if b % m == 0 and (b // m) * s >= 2048:
                best = m
        cap = getattr(self, "_pf_rows_cap", None)   # a micro-batch must fit the prefill P2P inbox
        while cap is not None and (b // best) * s > cap:
            best = next(m for m in range(best + 1, b + 1) if b % m == 0)
        return best

    def _prefill(self, b, s):
        m = self.prefill_microbatches(b, s)
        mb = b // m
        for d in self.drivers:
            if d.stage == 0:
                d.embed(b * s, prefill=True)
        for i in range(m):
            for d in self.drivers:
                for e in d.execs:
                    e.window(i * mb, mb, s)
                if d.stage > 0:
                    d.recv_hidden(mb * s)
                d.layers(mb * s, s)
                if d.stage < self.num_stages - 1:
                    d.send_hidden(mb * s)
                for e in d.execs:
                    e.window(0, 0, 0)
        for d in self.drivers:
            if d.stage == self.num_stages - 1:
                d.head(s)

    def _decode_compute(self, d: StageDriver, b):
        if d.stage == 0:
            d.embed(b, prefill=False)
        d.layers(b, 0)
        if d.stage == self.num_stages - 1:
            d.head(0)

    def _return_ids(self):
        if self.num_stages == 1:
            return
        for d in self.drivers:
            if d.stage == self.num_stages - 1:
                d.send_ids()
        for d in self.drivers:
            if d.stage == 0:
                d.recv_ids()

    def _decode_full(self, d: StageDriver, b):
        """One local stage's whole decode step in P2P mode: token ids in
        (stage 0) / out (last stage), hidden in, compute, hidden out -- all
        device-side, so it is captured as one graph per step."""
        if d.stage == self.num_stages - 1:
            d.send_ids()
        if d.stage == 0:
            d.recv_ids()
        if d.stage > 0:
            d.recv_hidden(b, decode=True)
        self._decode_compute(d, b)
        if d.stage < self.num_stages - 1:
            d.send_hidden(b, decode=True)

    def _decode_emulated_peer(self, b):
        """The whole pipeline's decode step on one GPU with the multi-GPU
        collective kernels (RankStreams): token ids back to stage 0 over the P2P
        link, then stage by stage with NVLink-style all-reduces and hand-offs."""
        self.sched.begin()
        if self.num_stages > 1:
            self.drivers[-1].send_ids()
            self.drivers[0].recv_ids()
        for d in self.drivers:
            if d.stage > 0:
                d.recv_hidden(b, decode=True)
            self._decode_compute(d, b)
            if d.stage < self.num_stages - 1:
                d.send_hidden(b, decode=True)
        self.sched.end()

    def _decode_step(self, b, graphs=None):
        if self.local_peer:
            if graphs is not None:
                graphs[0].replay()
                self._replayed += self._graph_launches[0]
            else:
                self._decode_emulated_peer(b)
            return
        if self._p2p:
            for i, d in enumerate(self.drivers):
                if graphs is not None:
                    graphs[i].replay()
                    self._replayed += self._graph_launches[i]
                else:
                    self._decode_full(d, b)
            return
        self._return_ids()
        for i, d in enumerate(self.drivers):
            if d.stage > 0:
                d.recv_hidden(b)
            if graphs is not None:
                graphs[i].replay()
                self._replayed += self._graph_launches[i]
            else:
                self._decode_compute(d, b)
            if d.stage < self.num_stages - 1:
                d.send_hidden(b)

    def _capture(self, b):
        """One CUDA graph per local stage for the decode compute (collectives
        inside; stage hand-offs stay outside on the same stream)."""
        key = b
        if key in self._graph_cache:   # one set of graphs per batch size served
            self._graphs, self._graph_launches = self._graph_cache[key]
            self._graph_key = key
            return self._graphs
        graphs, counts = [], []
        if self.local_peer:   # one graph over every emulated rank's stream (fork / join by events)
            g = torch.cuda.CUDAGraph()
            n0 = self._launch_count()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self._decode_emulated_peer(b)
            self._graphs, self._graph_key, self._graph_launches = [g], key, [self._launch_count() - n0]
            self._graph_cache[key] = (self._graphs, self._graph_launches)
            return self._graphs
        for d in self.drivers:
            g = torch.cuda.CUDAGraph()
            n0 = self._launch_count()
            # thread_local: the NCCL watchdog thread keeps querying events during capture
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                if self._p2p:
                    self._decode_full(d, b)
                else:
                    self._decode_compute(d, b)
            counts.append(self._launch_count() - n0)
            graphs.append(g)
        self._graphs, self._graph_key, self._graph_launches = graphs, key, counts
        self._graph_cache[key] = (graphs, counts)
        return graphs

    def _launch_count(self) -> int:
        fn = getattr(self.kernels, "launch_count", None)
        return fn() if fn else 0

    def _reset(self, b, s, s_out):
        for e in self.execs:
            e.kv.assign(b, s + s_out)
            if e.role.is_last:
                e.step.zero_()

    # ---------------------------------------------------------------- API
    def generate(self, prompt, output_len: int | None = None, return_logits: bool = False,
                 forced=None) -> GenerateResult:
        """Greedy generation (HF ``max_new_tokens`` semantics): the prefill
        emits token 1, then ``output_len - 1`` decode steps. ``prompt`` is a
        host int array [b, s_in]; returns host ids [b, output_len] on every
        rank (broadcast from the last stage under torch.distributed).
        ``forced`` [b, output_len] teacher-forces the token fed back to stage 0
        (the bf16-mode tolerance check); the returned ids stay the argmax."""
        if forced is not None:
            return_logits = True
            forced_dev = torch.as_tensor(np.asarray(forced, dtype=np.int32), device=self.device)
        prompt = np.asarray(prompt, dtype=np.int32)
        b, s = prompt.shape
        s_out = output_len or self.max_out
        if b > self.batch or s > self.max_prompt or s_out > self.max_out:
            raise InputError(f"request {(b, s, s_out)} exceeds engine shape "
                             f"{(self.batch, self.max_prompt, self.max_out)}")
        for e in self.execs:        # any batch up to the engine's: kernels run on the first b rows
            e.cur_b = b
        cuda = self.device.type == "cuda"
        if cuda and self.use_graphs and not return_logits:
            # warm the eager path once per batch size (kernel attributes, NCCL comms) before capture
            if b not in self._graph_cache:
                self._reset(b, s, s_out)
                for e in self.execs:
                    if e.role.is_first:
                        e.prompt[:b * s].copy_(torch.from_numpy(prompt.reshape(-1)))
                self._prefill(b, s)
                self._decode_step(b, None)
                torch.cuda.synchronize(self.device)
                self._capture(b)
        graphs = self._capture(b) if (cuda and self.use_graphs and not return_logits) else None
        self._replayed = 0
        n_launch0 = self._launch_count()
        self._reset(b, s, s_out)
        pin = torch.from_numpy(prompt.reshape(-1))
        if cuda:
            pin = pin.pin_memory()
        for e in self.execs:
            if e.role.is_first:
                e.prompt[:b * s].copy_(pin, non_blocking=True)
        logits = [] if return_logits else None
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if cuda else None
        t0 = ev() if cuda else None
        if cuda:
            t0.record()
        else:
            w0 = time.perf_counter()
        self._prefill(b, s)
        if return_logits:
            logits.append(self._gather_logits())
        if forced is not None:
            self._force(forced_dev, 0)
        step_ev = []
        if cuda:
            t1 = ev()
            t1.record()
        else:
            w1 = time.perf_counter()
        for t in range(1, s_out):
            if cuda:
                e0 = ev()
                e0.record()
            self._decode_step(b, graphs)
            if cuda:
                e1 = ev()
                e1.record()
                step_ev.append((e0, e1))
            if return_logits:
                logits.append(self._gather_logits())
            if forced is not None:
                self._force(forced_dev, t)
        if cuda:
            t2 = ev()
            t2.record()
        ids = self._collect_ids(b, s_out)
        if cuda:
            torch.cuda.synchronize(self.device)
            pre = t0.elapsed_time(t1) / 1e3
            dec = t1.elapsed_time(t2) / 1e3
            steps = [a.elapsed_time(c) for a, c in step_ev]
        else:
            w2 = time.perf_counter()
            pre, dec, steps = w1 - w0, w2 - w1, []
        lg = np.stack(logits, 0) if return_logits else None
        launches = self._launch_count() - n_launch0 + self._replayed
        return GenerateResult(ids, pre, dec, steps, lg, launches)

    def _force(self, forced_dev, t):
        for e in self._last_execs():
            e.ids[:forced_dev.shape[0]].copy_(forced_dev[:, t])

    def _last_execs(self):
        return [e for e in self.execs if e.role.is_last]

    def _gather_logits(self):
        last = sorted(self._last_execs(), key=lambda e: e.role.tp_rank)
        if not last:
            return None
        if len(last) == last[0].role.tp:
            return torch.cat([e.logits for e in last], dim=-1).float().cpu().numpy()
        return self.comm.gather_logits(last[0])

    def _collect_ids(self, b, s_out):
        last = self._last_execs()
        hist = last[0].history[:b, :s_out] if last else None
        return self.comm.broadcast_ids(hist, b, s_out, self.roles[-1].tp_group[0], self.device)

    def close(self):
        """Release the NVLink peer state (unmap peers' IPC buffers, free own
        ones, after a group barrier) and the captured graphs. Idempotent."""
        self._graphs = None
        self._graph_cache = {}
        links = {}
        for e in self.execs:
            if e.par is not None:
                e.par.close()
                e.par = None
            for link in list(e.p2p_send) + list(e.ids_send) + list(e.pf_send) + [e.p2p_recv, e.ids_recv, e.pf_recv]:
                if link is not None:
                    links[id(link)] = link      # an emulated link is held by both of its ends
            e.p2p_send, e.ids_send, e.p2p_recv, e.ids_recv = [], [], None, None
            e.pf_send, e.pf_recv = [], None
        for link in links.values():
            link.close()

    def service_time(self, task: TaskSpec, prompt=None) -> float:
        """Measured seconds for one request of this shape (the value the
        reference's ``service_times`` table holds, simulate.py:135-142)."""
        if prompt is None:
            rng = np.random.default_rng(1)
            prompt = rng.integers(0, self.cfg.vocab, size=(task.batch_size, task.input_len), dtype=np.int32)
        r = self.generate(prompt, task.output_len)
        return r.prefill_s + r.decode_s
