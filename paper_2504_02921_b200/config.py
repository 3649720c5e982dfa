"""Model / layout configuration, field-for-field with the reference.

ModelConfig mirrors model.py:38-67, LayoutConfig mirrors reranker.py:32-46
(same defaults, same invariants, same ConfigError messages).  PRESETS maps
BASELINE.json's configs onto them.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

PAD_ID = 0


@dataclass(frozen=True)
class ModelConfig:
    layers: int = 4
    model_dim: int = 128
    heads: int = 8
    kv_heads: int = 2
    head_dim: int = 16
    vocab_size: int = 32768
    rope_base: float = 10000.0
    max_position: int = 1024
    seed: int = 0
    # Architecture variants (the real bge-reranker-v2-gemma /
    # RankZephyr shapes).  Not in the reference; the defaults ARE the
    # reference model, so every parity statement holds unchanged for them.
    #   mlp          "gelu" (reference: gelu_tanh(x W_up) W_down, width 4d),
    #                "geglu" (Gemma) or "swiglu" (Mistral/Llama): gated, W_gate
    #                tensors named layers.{i}.mlp.w_gate
    #   ffn_dim      MLP width F (0 = 4 * model_dim)
    #   embed_scale  x = E[tok] * embed_scale (Gemma: sqrt(model_dim))
    #   attn_scale   softmax(scale * q.k) (real models: 1/sqrt(head_dim);
    #                folded into W_q on the device)
    mlp: str = "gelu"
    ffn_dim: int = 0
    embed_scale: float = 1.0
    attn_scale: float = 1.0

    @property
    def ffn(self) -> int:
        return self.ffn_dim or 4 * self.model_dim

    def validate(self) -> None:
        for name in ("layers", "model_dim", "heads", "kv_heads", "head_dim",
                     "vocab_size", "max_position"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.heads % self.kv_heads != 0:
            raise ConfigError(
                f"heads ({self.heads}) must be divisible by kv_heads ({self.kv_heads})")
        if self.model_dim != self.heads * self.head_dim:
            raise ConfigError(
                f"model_dim ({self.model_dim}) != heads*head_dim "
                f"({self.heads * self.head_dim})")
        if self.rope_base <= 0:
            raise ConfigError("rope_base must be positive")
        if self.mlp not in ("gelu", "geglu", "swiglu"):
            raise ConfigError(f"mlp must be gelu, geglu or swiglu, got {self.mlp!r}")
        if self.ffn_dim < 0 or (self.mlp != "gelu" and self.ffn % 32):
            raise ConfigError(f"ffn_dim {self.ffn_dim} invalid (gated MLPs need a multiple of 32)")
        if not (self.embed_scale > 0 and self.attn_scale > 0):
            raise ConfigError("embed_scale and attn_scale must be positive")

    @property
    def group_size(self) -> int:
        return self.heads // self.kv_heads


@dataclass(frozen=True)
class LayoutConfig:
    document_len: int = 256
    query_len: int = 48
    pad_id: int = PAD_ID

    def validate(self) -> None:
        if self.document_len < 1 or self.query_len < 1:
            raise ConfigError("document_len and query_len must be >= 1")
        if self.pad_id != 0:
            raise ConfigError("pad id 0 is reserved and fixed")

    @property
    def total_len(self) -> int:
        return self.document_len + self.query_len


# BASELINE.json configs.  The MLP stays the reference's
# GELU 4*d (model.py:172-173); only the widths/depths take the named shapes.
PRESETS = {
    "c1_tiny": (ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                            vocab_size=32768, seed=0),
                LayoutConfig(document_len=128, query_len=48)),
    "c2_gemma2b": (ModelConfig(layers=18, model_dim=2048, heads=8, kv_heads=1, head_dim=256,
                               vocab_size=256000, seed=0),
                   LayoutConfig(document_len=512, query_len=48)),
    "c3_mistral7b": (ModelConfig(layers=32, model_dim=4096, heads=32, kv_heads=8, head_dim=128,
                                 vocab_size=32000, seed=0),
                     LayoutConfig(document_len=512, query_len=48)),
    "c5_mistral7b_d2048": (ModelConfig(layers=32, model_dim=4096, heads=32, kv_heads=8,
                                       head_dim=128, vocab_size=32000, max_position=4096,
                                       seed=0),
                           LayoutConfig(document_len=2048, query_len=48)),
    # f4: the true architectures of the named shapes (outside reference parity)
    "c2_gemma2b_real": (ModelConfig(layers=18, model_dim=2048, heads=8, kv_heads=1,
                                    head_dim=256, vocab_size=256000, seed=0, mlp="geglu",
                                    ffn_dim=16384, embed_scale=2048 ** 0.5,
                                    attn_scale=256 ** -0.5),
                        LayoutConfig(document_len=512, query_len=48)),
    "c3_mistral7b_real": (ModelConfig(layers=32, model_dim=4096, heads=32, kv_heads=8,
                                      head_dim=128, vocab_size=32000, seed=0, mlp="swiglu",
                                      ffn_dim=14336, attn_scale=128 ** -0.5),
                          LayoutConfig(document_len=512, query_len=48)),
}
