"""Llama-style decoder configuration: a superset of the reference ``ModelSpec``.

The reference model document carries only ``num_layers``, ``hidden_dim`` and
``bytes_per_param`` (reference ``pkg/src/heteroplan/cluster.py:223-260``) and
ignores unknown keys, so the superset written by ``to_model_dict`` stays
loadable by the reference planner while carrying what the data path needs
(heads, kv heads, intermediate, vocab, eps, rope theta).

Shapes: SURVEY.md §8 table (Llama-2 7B/13B/70B and the tiny C1 config,
intermediate 768 / vocab 32000 fixed per SURVEY Appendix B #1).
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, replace
from typing import Mapping

from .plan import InputError, ModelSpec


@dataclass(frozen=True)
class LlamaConfig:
    name: str
    num_layers: int
    hidden_dim: int
    num_heads: int
    num_kv_heads: int
    intermediate: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0
    bytes_per_param: int = 2
    head_dim_override: int = 0   # 0: hidden_dim // num_heads (a TP shard viewed as a model sets it)

    def __post_init__(self):
        if self.hidden_dim % self.num_heads:
            raise InputError("hidden_dim must divide by num_heads")
        if self.num_heads % self.num_kv_heads:
            raise InputError("num_heads must divide by num_kv_heads")

    @property
    def head_dim(self) -> int:
        return self.head_dim_override or self.hidden_dim // self.num_heads

    @property
    def group(self) -> int:
        return self.num_heads // self.num_kv_heads

    @property
    def qkv_out(self) -> int:
        return (self.num_heads + 2 * self.num_kv_heads) * self.head_dim

    def params_per_layer(self) -> int:
        H, hd = self.hidden_dim, self.head_dim
        return (H * self.num_heads * hd + 2 * H * self.num_kv_heads * hd
                + self.num_heads * hd * H + 3 * H * self.intermediate + 2 * H)

    def to_model_spec(self) -> ModelSpec:
        return ModelSpec(self.num_layers, self.hidden_dim, self.bytes_per_param)

    def to_model_dict(self) -> dict:
        d = asdict(self)
        d["schema_version"] = 1
        return d

    def check_tp(self, tp: int) -> None:
        """Megatron column/row split needs every sharded dim to divide by TP."""
        for what, n in (("num_heads", self.num_heads), ("num_kv_heads", self.num_kv_heads),
                        ("intermediate", self.intermediate), ("vocab", self.vocab)):
            if n % tp:
                raise InputError(f"{what}={n} is not divisible by tp={tp}")


TINY = LlamaConfig("tiny", 4, 256, 8, 8, 768, 32000, bytes_per_param=4)
LLAMA2_7B = LlamaConfig("llama2-7b", 32, 4096, 32, 32, 11008, 32000)
LLAMA2_13B = LlamaConfig("llama2-13b", 40, 5120, 40, 40, 13824, 32000)
LLAMA2_70B = LlamaConfig("llama2-70b", 80, 8192, 64, 8, 28672, 32000)

PRESETS = {c.name: c for c in (TINY, LLAMA2_7B, LLAMA2_13B, LLAMA2_70B)}


def preset(name: str, **overrides) -> LlamaConfig:
    if name not in PRESETS:
        raise InputError(f"unknown model preset {name!r}; have {sorted(PRESETS)}")
    return replace(PRESETS[name], **overrides) if overrides else PRESETS[name]


def config_from_dict(doc: Mapping) -> LlamaConfig:
    """Read a model document. A reference-only document (three keys) is
    completed from the preset whose hidden/layers match."""
    try:
        if "num_heads" not in doc:
            for c in PRESETS.values():
                if c.hidden_dim == int(doc["hidden_dim"]) and c.num_layers == int(doc["num_layers"]):
                    return replace(c, bytes_per_param=int(doc["bytes_per_param"]))
            raise InputError("model document lacks num_heads and matches no preset")
        return LlamaConfig(
            name=str(doc.get("name", "custom")),
            num_layers=int(doc["num_layers"]), hidden_dim=int(doc["hidden_dim"]),
            num_heads=int(doc["num_heads"]),
            num_kv_heads=int(doc.get("num_kv_heads", doc["num_heads"])),
            intermediate=int(doc["intermediate"]), vocab=int(doc.get("vocab", 32000)),
            rms_eps=float(doc.get("rms_eps", 1e-5)), rope_theta=float(doc.get("rope_theta", 1e4)),
            bytes_per_param=int(doc["bytes_per_param"]))
    except InputError:
        raise
    except (KeyError, TypeError, ValueError) as exc:
        raise InputError(f"bad model document: {exc}") from exc


def load_model_config(path) -> LlamaConfig:
    with open(path) as fh:
        try:
            return config_from_dict(json.load(fh))
        except json.JSONDecodeError as exc:
            raise InputError(f"{path}: {exc}") from exc
