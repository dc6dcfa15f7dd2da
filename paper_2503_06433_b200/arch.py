"""LLaMA architecture constants the reference's ModelSpec cannot carry.

The reference's ModelSpec YAML rejects unknown keys (specs.py:342-344), so
hidden size, FFN width, vocabulary and RoPE base live in this separate
document; :meth:`LlamaArch.model_spec` derives the reference ModelSpec with
``params_per_layer`` folded as total/L so ``total_weight_bytes`` is exact
(SURVEY.md Appendix A.1).
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass
from pathlib import Path
from typing import Any, Mapping

import yaml

from .specs import ConfigError, ModelSpec


@dataclass(frozen=True)
class LlamaArch:
    name: str
    num_layers: int
    hidden: int
    num_query_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5

    def __post_init__(self) -> None:
        for f in ("num_layers", "hidden", "num_query_heads", "num_kv_heads", "head_dim", "ffn", "vocab"):
            v = getattr(self, f)
            if not isinstance(v, int) or v <= 0:
                raise ConfigError(f"LlamaArch.{f} must be a positive integer")
        if self.num_query_heads % self.num_kv_heads:
            raise ConfigError("num_query_heads must be a multiple of num_kv_heads")
        if self.head_dim % 64:
            raise ConfigError("head_dim must be a multiple of 64 (128-byte K/V rows)")
        if self.ffn % 32 or self.hidden % 64:
            raise ConfigError("ffn must be a multiple of 32 and hidden of 64")

    @property
    def group(self) -> int:
        return self.num_query_heads // self.num_kv_heads

    @property
    def qkv_dim(self) -> int:
        return (self.num_query_heads + 2 * self.num_kv_heads) * self.head_dim

    def params_per_layer_exact(self) -> int:
        h, d = self.hidden, self.head_dim
        return h * self.qkv_dim + self.num_query_heads * d * h + 3 * h * self.ffn + 2 * h

    def embed_head_params(self) -> int:
        return 2 * self.vocab * self.hidden + self.hidden

    def total_params(self) -> int:
        return self.num_layers * self.params_per_layer_exact() + self.embed_head_params()

    def model_spec(self, bytes_per_param: int = 2) -> ModelSpec:
        return ModelSpec(
            num_layers=self.num_layers,
            params_per_layer=math.ceil(self.total_params() / self.num_layers),
            num_query_heads=self.num_query_heads,
            num_kv_heads=self.num_kv_heads,
            head_dim=self.head_dim,
            bytes_per_param=bytes_per_param,
        )

    def validate_layout(self, tp: int, pp: int) -> None:
        if self.num_layers % pp:
            raise ConfigError(f"pp={pp} does not divide num_layers={self.num_layers}")
        if self.num_kv_heads % tp:
            raise ConfigError(f"tp={tp} does not divide num_kv_heads={self.num_kv_heads}")
        if self.vocab % tp or (self.vocab // tp) % 8:
            raise ConfigError(f"tp={tp} must split the vocabulary into multiples of 8")
        if (self.ffn // tp) % 32 or self.ffn % tp:
            raise ConfigError(f"tp={tp} must split ffn into multiples of 32")

    def as_dict(self) -> dict[str, Any]:
        return asdict(self)


PRESETS: dict[str, LlamaArch] = {
    # BASELINE.json configs[0]: 2 layers, hidden 256, 4 heads (h_q = h_kv = 4)
    "tiny": LlamaArch("tiny", 2, 256, 4, 4, 64, 768, 1024, rope_theta=10000.0),
    # GQA variant of the tiny config (one KV head per rank at TP=2)
    "tiny-gqa": LlamaArch("tiny-gqa", 2, 256, 4, 2, 64, 768, 1024, rope_theta=10000.0),
    "llama3-8b": LlamaArch("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256, rope_theta=500000.0),
    "llama2-13b": LlamaArch("llama2-13b", 40, 5120, 40, 40, 128, 13824, 32000, rope_theta=10000.0),
    "llama3-70b": LlamaArch("llama3-70b", 80, 8192, 64, 8, 128, 28672, 128256, rope_theta=500000.0),
}


def arch_from_mapping(doc: Mapping[str, Any]) -> LlamaArch:
    allowed = set(LlamaArch.__dataclass_fields__)
    extra = set(doc) - allowed
    if extra:
        raise ConfigError(f"unknown LlamaArch fields: {sorted(extra)}")
    return LlamaArch(**doc)


def load_arch(path: str | Path) -> LlamaArch:
    with open(path, "r", encoding="utf-8") as fh:
        doc = yaml.safe_load(fh)
    if not isinstance(doc, dict):
        raise ConfigError(f"{path}: expected a mapping")
    return arch_from_mapping(doc)
