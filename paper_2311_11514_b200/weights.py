"""Seeded random-init weights and Megatron sharding of them.

Random init per SURVEY §8c: normal(0, 0.02) for every matrix; RMSNorm gains
1 + normal(0, 0.02) (not exactly 1, so a dropped gain is visible in parity).
Every tensor draws from its own ``numpy.random.Generator(PCG64)`` stream
keyed by ``[seed, layer + 1, tensor_code]`` (layer 0 for the global tensors),
so any rank can materialise just its own layers and two processes that ask
for the same tensor get the same bits. Names follow HF ``LlamaForCausalLM``
state-dict keys so the CPU oracle can be pinned against transformers.

Sharding (the plan's stage j, TP rank r of t):
  * q/k/v/gate/up are column-parallel: rows [r*n/t, (r+1)*n/t) of the
    [out, in] matrix (per head for q/k/v);
  * o/down are row-parallel: columns [r*n/t, (r+1)*n/t);
  * lm_head is vocab-parallel: rows [r*V/t, (r+1)*V/t);
  * embedding and norms are replicated.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .config import LlamaConfig

_CODES = {"embed": 1, "norm": 2, "lm_head": 3,
          "q": 10, "k": 11, "v": 12, "o": 13, "gate": 14, "up": 15, "down": 16,
          "ln_attn": 17, "ln_mlp": 18}

LAYER_TENSORS = ("q", "k", "v", "o", "gate", "up", "down", "ln_attn", "ln_mlp")


def tensor_shape(cfg: LlamaConfig, name: str) -> tuple[int, ...]:
    H, hd = cfg.hidden_dim, cfg.head_dim
    return {
        "embed": (cfg.vocab, H), "norm": (H,), "lm_head": (cfg.vocab, H),
        "q": (cfg.num_heads * hd, H), "k": (cfg.num_kv_heads * hd, H),
        "v": (cfg.num_kv_heads * hd, H), "o": (H, cfg.num_heads * hd),
        "gate": (cfg.intermediate, H), "up": (cfg.intermediate, H),
        "down": (H, cfg.intermediate), "ln_attn": (H,), "ln_mlp": (H,),
    }[name]


def init_tensor(cfg: LlamaConfig, seed: int, name: str, layer: int = -1) -> np.ndarray:
    """fp32 host tensor; identical bits for identical (seed, layer, name)."""
    rng = np.random.default_rng([seed, layer + 1, _CODES[name]])
    shape = tensor_shape(cfg, name)
    x = rng.standard_normal(size=shape, dtype=np.float32)
    x *= np.float32(0.02)
    if name in ("norm", "ln_attn", "ln_mlp"):
        x += np.float32(1.0)
    return x


def _workers() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def layer_stream(cfg: LlamaConfig, seed: int, layers, lookahead: int = 2):
    """Yield ``(l, {name: fp32 tensor})`` for ``layers`` in order, the tensors
    drawn by a thread pool (numpy's generators release the GIL while filling)
    up to ``lookahead`` layers ahead. Same bits as ``init_tensor``: every tensor
    keeps its own seeded stream, only the wall time changes (7B: ~140 s of
    single-threaded draws)."""
    layers = list(layers)
    with ThreadPoolExecutor(_workers()) as ex:
        pending = {}

        def submit(i):
            if i < len(layers) and i not in pending:
                pending[i] = {n: ex.submit(init_tensor, cfg, seed, n, layers[i]) for n in LAYER_TENSORS}

        for i in range(min(lookahead + 1, len(layers))):
            submit(i)
        for i, l in enumerate(layers):
            submit(i + lookahead)
            futs = pending.pop(i)
            yield l, {n: f.result() for n, f in futs.items()}


def init_globals(cfg: LlamaConfig, seed: int, names) -> dict:
    """The non-layer tensors (embed / norm / lm_head), drawn in parallel."""
    with ThreadPoolExecutor(_workers()) as ex:
        futs = {n: ex.submit(init_tensor, cfg, seed, n) for n in names}
        return {n: f.result() for n, f in futs.items()}


def init_host_weights(cfg: LlamaConfig, seed: int = 0, layers=None,
                      with_embed: bool = True, with_head: bool = True) -> dict:
    """{"embed", "norm", "lm_head", "layers": [ {q,k,v,o,...}, ... ]} fp32."""
    layers = range(cfg.num_layers) if layers is None else layers
    names = (["embed"] if with_embed else []) + (["norm", "lm_head"] if with_head else [])
    w = dict(init_globals(cfg, seed, names))
    w["layers"] = {}
    for l, lw in layer_stream(cfg, seed, layers):
        w["layers"][l] = lw
    return w


def to_hf_state_dict(cfg: LlamaConfig, w: dict) -> dict:
    """HF LlamaForCausalLM key names (used only to pin the oracle)."""
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["norm"],
          "lm_head.weight": w["lm_head"]}
    names = {"q": "self_attn.q_proj", "k": "self_attn.k_proj", "v": "self_attn.v_proj",
             "o": "self_attn.o_proj", "gate": "mlp.gate_proj", "up": "mlp.up_proj",
             "down": "mlp.down_proj", "ln_attn": "input_layernorm",
             "ln_mlp": "post_attention_layernorm"}
    for l, lw in w["layers"].items():
        for k, v in lw.items():
            sd[f"model.layers.{l}.{names[k]}.weight"] = v
    return sd


def shard_rows(x: np.ndarray, rank: int, tp: int) -> np.ndarray:
    n = x.shape[0] // tp
    return x[rank * n:(rank + 1) * n]


def shard_cols(x: np.ndarray, rank: int, tp: int) -> np.ndarray:
    n = x.shape[1] // tp
    return x[:, rank * n:(rank + 1) * n]


def shard_layer(cfg: LlamaConfig, lw: dict, rank: int, tp: int) -> dict:
    """Per-rank fused tensors the kernels consume:
    ``wqkv`` [(hq+2hkv)/t*hd, H] = cat(q_r, k_r, v_r); ``wo`` [H, hq/t*hd];
    ``wgu`` [2I/t, H] = cat(gate_r, up_r); ``wdown`` [H, I/t]; two gains."""
    cfg.check_tp(tp)
    return {
        "wqkv": np.ascontiguousarray(np.concatenate(
            [shard_rows(lw["q"], rank, tp), shard_rows(lw["k"], rank, tp),
             shard_rows(lw["v"], rank, tp)], axis=0)),
        "wo": np.ascontiguousarray(shard_cols(lw["o"], rank, tp)),
        "wgu": np.ascontiguousarray(np.concatenate(
            [shard_rows(lw["gate"], rank, tp), shard_rows(lw["up"], rank, tp)], axis=0)),
        "wdown": np.ascontiguousarray(shard_cols(lw["down"], rank, tp)),
        "ln_attn": lw["ln_attn"], "ln_mlp": lw["ln_mlp"],
    }


def synthetic_prompts(cfg: LlamaConfig, batch: int, input_len: int, seed: int = 1) -> np.ndarray:
    """Uniform token ids over [0, V) (SURVEY §8c prompts, seed 1)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, cfg.vocab, size=(batch, input_len), dtype=np.int64).astype(np.int32)
