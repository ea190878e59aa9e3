"""Layer-group geometries of the BASELINE.json configs, expressed in the
reference's model-config vocabulary (reference proj/configs/*.cfg) with the
bytes derived from heads/dtype (bptl = 2*Hkv*D*e for attention;
Mamba groups carry their per-layer state bytes with tokens_per_page = 1,
simulator.cpp:222-244).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import torch

from .jenga import LayerGroupSpec, LayerKind, ModelSpec

_DTYPE_BYTES = {torch.float32: 4, torch.bfloat16: 2, torch.float16: 2}


@dataclass
class GroupGeometry:
    name: str
    kind: LayerKind
    num_layers: int
    num_kv_heads: int = 0
    num_q_heads: int = 0
    head_dim: int = 0
    dtype: torch.dtype = torch.bfloat16
    tokens_per_page: int = 16
    window: int = 0
    state_bytes: int = 0           # mamba: bytes of one layer's state; vision: embedding bytes per token
    checkpoint_interval: int = 512

    @property
    def is_attention(self) -> bool:
        return self.kind in (LayerKind.kFullAttention, LayerKind.kSlidingWindow, LayerKind.kCrossAttention)

    @property
    def bytes_per_token_per_layer(self) -> int:
        if self.kind in (LayerKind.kMamba, LayerKind.kVisionEmbedding):
            return self.state_bytes
        return 2 * self.num_kv_heads * self.head_dim * _DTYPE_BYTES[self.dtype]

    def group_spec(self) -> LayerGroupSpec:
        return LayerGroupSpec(
            name=self.name, kind=self.kind, num_layers=self.num_layers,
            bytes_per_token_per_layer=self.bytes_per_token_per_layer,
            tokens_per_page=1 if self.kind == LayerKind.kMamba else self.tokens_per_page,
            window_tokens=self.window if self.kind == LayerKind.kSlidingWindow else 0,
            checkpoint_interval_tokens=self.checkpoint_interval if self.kind == LayerKind.kMamba else 0)


@dataclass
class ModelGeometry:
    name: str
    groups: List[GroupGeometry] = field(default_factory=list)
    softcap: float = 0.0

    def spec(self) -> ModelSpec:
        return ModelSpec(self.name, [g.group_spec() for g in self.groups])

    def group_index(self, name: str) -> int:
        for i, g in enumerate(self.groups):
            if g.name == name:
                return i
        raise KeyError(name)


def toy(tokens_per_page: int = 16) -> ModelGeometry:
    """configs[0]: Gemma-2-style 2 layers (1 full + 1 SWA-512), Hkv=8, D=128, fp32."""
    f32 = torch.float32
    return ModelGeometry("toy-gemma2-2layer", [
        GroupGeometry("full", LayerKind.kFullAttention, 1, 8, 16, 128, f32, tokens_per_page),
        GroupGeometry("window", LayerKind.kSlidingWindow, 1, 8, 16, 128, f32, tokens_per_page, window=512),
    ])


def gemma2_9b(tokens_per_page: int = 16, softcap: float = 50.0) -> ModelGeometry:
    """configs[1]: Gemma-2-9B — 42 layers alternating full / SWA-4096,
    Hq=16, Hkv=8, D=256, bf16, attention-logit soft-capping at 50 (the
    model's attn_logit_softcapping)."""
    bf = torch.bfloat16
    return ModelGeometry("gemma2-9b", [
        GroupGeometry("full", LayerKind.kFullAttention, 21, 8, 16, 256, bf, tokens_per_page),
        GroupGeometry("window", LayerKind.kSlidingWindow, 21, 8, 16, 256, bf, tokens_per_page, window=4096),
    ], softcap=softcap)


def jamba_style(tokens_per_page: int = 16) -> ModelGeometry:
    """configs[2]: 4 attention layers (Hq=32, Hkv=8, D=128, bf16) + 28 Mamba
    layers whose fp32 state is (8192*3 + 8192*16)*4 = 622,592 B per layer."""
    bf = torch.bfloat16
    return ModelGeometry("jamba-style", [
        GroupGeometry("attn", LayerKind.kFullAttention, 4, 8, 32, 128, bf, tokens_per_page),
        GroupGeometry("ssm", LayerKind.kMamba, 28, state_bytes=(8192 * 3 + 8192 * 16) * 4, checkpoint_interval=512),
    ])


def llama32_11b_vision(tokens_per_page: int = 16) -> ModelGeometry:
    """configs[3]: 32 self-attention + 8 cross-attention layers over image KV,
    Hq=32, Hkv=8, D=128, bf16."""
    bf = torch.bfloat16
    return ModelGeometry("llama-3.2-11b-vision", [
        GroupGeometry("self", LayerKind.kFullAttention, 32, 8, 32, 128, bf, tokens_per_page),
        GroupGeometry("cross", LayerKind.kCrossAttention, 8, 8, 32, 128, bf, tokens_per_page),
    ])


MODELS = {"toy": toy, "gemma2-9b": gemma2_9b, "jamba-style": jamba_style,
          "llama-3.2-11b-vision": llama32_11b_vision}
